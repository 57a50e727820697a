"""One line per bench JSON in a log (lines starting with '==' name the run)."""
import json
import sys

name = None
for line in open(sys.argv[1]):
    if line.startswith("=="):
        name = line.strip()
    elif line.startswith("{"):
        d = json.loads(line)
        c = d.get("comm_us") or {}
        head = [name, "%.4f ms" % d["value"], "local %.1f us" % d["roofline"]["launch_us"],
                "frac %.3f" % d["roofline"]["frac"]]
        if "reduced_phase_us" in c:
            r = c.get("per_round_median_us", {})
            head.append("reduced %.1f us (p2p %.1f, window %.1f; rounds y %.1f steps %s x %.1f)" % (
                c["reduced_phase_us"], c["p2p_kernel_us"], c["window_kernel_us"], r.get("y_exchange", -1),
                [round(v, 1) for v in r.get("schedule_steps", [])], r.get("x_exchange", -1)))
        elif "fused_reduced_kernel_us" in c:
            head.append("fused reduced %.1f us" % c["fused_reduced_kernel_us"])
        elif c.get("fused_into_tile_kernel"):
            head.append("reduced phase fused into the tile kernel")
        elif c:
            head.append("y %.1f st %s x %.1f back %.1f" % (
                c.get("y_exchange", 0), [round(v, 1) for v in c.get("stages", [])],
                c.get("x_exchange", 0), c.get("backsub_kernel", 0)))
        print(" ".join(str(h) for h in head))
