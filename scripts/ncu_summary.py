"""Summarise an .ncu-rep: duration, DRAM bytes/throughput, occupancy, grid, top stall reasons."""
import csv
import io
import json
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    return [dict(zip(h, r)) for r in rows[2:]], dict(zip(h, units))


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return None


def summarise(rep):
    kernels, units = raw(rep)
    res = []
    for d in kernels:
        st = {k: num(v) for k, v in d.items() if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}
        st = {k: v for k, v in st.items() if v}
        tot = sum(st.values()) or 1
        top = sorted(st.items(), key=lambda z: -z[1])[:8]
        dur = num(d.get("gpu__time_duration.sum"))
        rd = num(d.get("dram__bytes_read.sum"))
        wr = num(d.get("dram__bytes_write.sum"))
        u_dur = units.get("gpu__time_duration.sum")
        u_b = units.get("dram__bytes_read.sum")
        scale_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                   "GB": 1e9}.get(u_b, 1)
        scale_t = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9,
                   "us": 1e-6, "ms": 1e-3, "s": 1}.get(u_dur, 1)
        res.append({
            "kernel": d.get("Kernel Name", "")[:80],
            "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
            "cluster": d.get("launch__cluster_dim_x") or d.get("launch__cluster_size"),
            "regs": d.get("launch__registers_per_thread"),
            "duration_s": dur * scale_t if dur else None,
            "dram_read_bytes": rd * scale_b if rd else None,
            "dram_write_bytes": wr * scale_b if wr else None,
            "dram_GBps": ((rd + wr) * scale_b / (dur * scale_t) / 1e9) if (rd and wr and dur) else None,
            "dram_pct_peak": num(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")),
            "units": {"duration": u_dur, "bytes": u_b},
            "achieved_occupancy": num(d.get("sm__warps_active.avg.pct_of_peak_sustained_active")),
            "stalls_pct": {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): round(100 * v / tot, 1) for k, v in top},
        })
    return res


if __name__ == "__main__":
    for r in summarise(sys.argv[1]):
        print(json.dumps(r, indent=1))
