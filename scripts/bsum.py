"""One line per bench JSON line in the given logs (value, tile-kernel us, frac, clocks)."""
import json
import sys
for f in sys.argv[1:]:
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            r = d.get("roofline") or {}
            print(f, d["value"], r.get("launch_us"), r.get("frac"), d.get("clocks"), d.get("gpu_launches"), d.get("comm_us"))
        elif "trace" in l:
            print("   ", l.strip()[:400])
