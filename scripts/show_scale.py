import json
import sys

name = None
for line in open(sys.argv[1]):
    if line.startswith("=="):
        name = line.strip()
    elif line.startswith("{"):
        d = json.loads(line)
        c = d.get("comm_us") or {}
        if "fused_reduced_kernel_us" in c:
            print(name, "%.4f ms" % d["value"], "local %.1f us" % d["roofline"]["launch_us"],
                  "frac %.3f" % d["roofline"]["frac"], "fused reduced %.1f us" % c["fused_reduced_kernel_us"])
            continue
        print(name, "%.4f ms" % d["value"], "local %.1f us" % d["roofline"]["launch_us"],
              "frac %.3f" % d["roofline"]["frac"], "y %.1f st %s x %.1f back %.1f" % (
                  c.get("y_exchange", 0), [round(v, 1) for v in c.get("stages", [])],
                  c.get("x_exchange", 0), c.get("backsub_kernel", 0)) if c else "")
