"""Copy the ncu summaries of scripts/profile_round.sh from gpurun_out/ into profiles/ and refresh
profiles/ncu_traffic.json (DRAM read + write bytes per launch of each config's dominant kernel)
and the launch list of the cfg2 step."""
import csv
import json
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"


def objects(path):
    txt = open(path).read()
    dec, i, res = json.JSONDecoder(), 0, []
    while i < len(txt):
        while i < len(txt) and txt[i] in " \n\r\t":
            i += 1
        if i >= len(txt):
            break
        o, i = dec.raw_decode(txt, i)
        res.append(o)
    return res


traffic_keys = {"cfg2": "cfg2_p1", "cfg4d2": "cfg4_d2_p1", "cfg5": "cfg5_p1", "cfg3": "cfg3_p1"}
tpath = os.path.join(PROF, "ncu_traffic.json")
traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
for name in ("cfg2", "cfg4d2", "cfg5", "cfg3", "penta"):
    src = os.path.join(OUT, f"sum_{name}.json")
    if not os.path.exists(src):
        continue
    objs = objects(src)
    json.dump(objs, open(os.path.join(PROF, f"{tag}_ncu_{name}_final.json"), "w"), indent=1)
    tile = [o for o in objs if o["kernel"].startswith("void k_tile")]
    if tile and name in traffic_keys:
        o = tile[0]
        traffic[traffic_keys[name]] = (o["dram_read_bytes"] or 0) + (o["dram_write_bytes"] or 0)
traffic["_source"] = ("dram__bytes_read.sum + dram__bytes_write.sum of the k_tile launch in one "
                      f"ncu --set full capture (profiles/{tag}_ncu_*_final.json), bytes per launch")
json.dump(traffic, open(tpath, "w"), indent=1)

lpath = os.path.join(OUT, "launches_cfg2.csv")
if os.path.exists(lpath):
    rows = [r for r in csv.reader(l for l in open(lpath) if l.startswith('"'))]
    h = rows[0]
    agg = OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"]
        k = k.split("(")[0] if not k.startswith("void at::") else k[:60]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"].replace(",", "")) / 1e3
    res = {"source": "ncu --metrics gpu__time_duration.sum --clock-control none, python bench.py "
                     "--steps 5 --warmup 3 (cfg2, N=1); cold-cache serialised launches",
           "kernels": [{"kernel": k, "launches": n, "total_us": round(t, 1), "per_launch_us": round(t / n, 1)}
                       for k, (n, t) in agg.items()]}
    json.dump(res, open(os.path.join(PROF, f"{tag}_launches_cfg2_p1.json"), "w"), indent=1)
print(json.dumps(traffic, indent=1))
