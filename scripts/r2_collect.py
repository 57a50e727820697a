"""Copy the round-2 ncu summaries of scripts/r2_profile.sh (gpurun_out/r2p_*) into profiles/:
r2_ncu_<cfg>.json + hotspots, the launch lists (r2_launches.json) and the per-launch DRAM
traffic used by bench.py's roofline.traffic (ncu_traffic.json)."""
import csv
import io
import json
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def first_json(path):
    txt = open(path).read()
    return json.JSONDecoder().raw_decode(txt, txt.index("{"))[0]


traffic_path = os.path.join(PROF, "ncu_traffic.json")
traffic = json.load(open(traffic_path))
for name, key in (("cfg2", "cfg2_p1"), ("penta", "penta_p1"), ("cfg5", "cfg5_p1")):
    src = os.path.join(OUT, f"r2p_ncu_{name}_sum.json")
    if not os.path.exists(src):
        continue
    d = first_json(src)
    json.dump(d, open(os.path.join(PROF, f"r2_ncu_{name}.json"), "w"), indent=1)
    shutil.copy(os.path.join(OUT, f"r2p_ncu_{name}_hot.txt"), os.path.join(PROF, f"r2_ncu_{name}_hotspots.txt"))
    traffic[key] = d["dram_read_bytes"] + d["dram_write_bytes"]
traffic["_source"] = ("dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel in one ncu --set full "
                      "capture per launch (round 2, end of round: profiles/r2_ncu_cfg2.json, r2_ncu_cfg5.json, "
                      "r2_ncu_penta.json; round 1 for the others)")
json.dump(traffic, open(traffic_path, "w"), indent=0)

launches = {"_source": "ncu --metrics gpu__time_duration.sum --clock-control none (scripts/r2_profile.sh), "
                       "cold-cache serialised launches of bench.py --no-graph; compare shares, not absolutes"}
for name in ("cfg2", "penta", "cfg5"):
    src = os.path.join(OUT, f"r2p_launches_{name}.csv")
    if not os.path.exists(src):
        continue
    lines = [l for l in open(src) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    launches[name] = [{"kernel": r["Kernel Name"].split("(")[0], "duration": float(r["Metric Value"]),
                       "unit": r["Metric Unit"]} for r in rows if r["Metric Name"] == "gpu__time_duration.sum"]
json.dump(launches, open(os.path.join(PROF, "r2_launches.json"), "w"), indent=1)
print({k: len(v) for k, v in launches.items() if k != "_source"}, {k: traffic[k] for k in traffic if k != "_source"})
