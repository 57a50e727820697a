"""Top SASS lines by warp-stall samples (with a few lines of context) from an .ncu-rep."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:]]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[key] or 0) for d in data) or 1
order = sorted(range(len(data)), key=lambda i: -float(data[i][key] or 0))[:n]
for i in order:
    print("---- %.1f%%" % (100 * float(data[i][key]) / tot))
    for d in data[max(0, i - 4):i + 2]:
        print("%5.1f%% %s %s" % (100 * float(d[key] or 0) / tot, d["Address"][-5:], d["Source"][:95]))
