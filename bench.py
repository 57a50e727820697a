#!/usr/bin/env python
"""Benchmark: ms per 8192x256^2 fp64 cyclic tridiagonal solve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl reference]

N = 1 runs in-process; N > 1 must be launched with torchrun (one rank per GPU, NCCL).
The workload is BASELINE.json configs[1] (strong scaling): the global 8192x256x256 grid,
bands B[1/3,1,1/3], cyclic, solved along index 0 and split into N equal slabs (P:5).
A "step" is one ctri_solve (all of (a1)-(a4)) on inputs resident in HBM; timing uses
CUDA events on the solve stream between barrier+synchronize brackets, max over ranks.
Each array is 4.3 GB/N (> 126 MB L2 for every N <= 8), so no L2 flush is needed.

Rank 0 prints ONE JSON line (keys per the driver contract, plus roofline / cpu_baseline /
e2e / clocks / per-stage communication times).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms per 8192×256² fp64 cyclic-tridiag solve, % HBM roofline, at 1/2/4/8 B200"
BYTES_PER_POINT = 16  # algorithmic: read b once, write x once (fp64)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="cfg2",
                    choices=["cfg1", "cfg2", "cfg3", "cfg4_d1", "cfg4_d2", "cfg5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dims", default=None, help="override: global dims N0,N1,N2 (measurement)")
    ap.add_argument("--sd", type=int, default=0, help="solve dim with --dims")
    ap.add_argument("--scheme", default="collocated",
                    choices=["collocated", "staggered_deriv", "staggered_interp"],
                    help="cfg5 compact scheme: collocated derivative (P:65-67) or the staggered "
                         "sixth-order derivative / interpolation (P:202-206)")
    ap.add_argument("--reduced", default="pcr", choices=["pcr", "fused", "allgather", "nccl"],
                    help="nparts > 1 reduced system: the P2P pairwise schedule kernel + window pass "
                         "(default), fused into the tile kernel (opt-in), the P2P all-gather with "
                         "A^-1 rows (N4), or host-issued NCCL rounds")
    ap.add_argument("--penta", action="store_true",
                    help="pentadiagonal system (r = 2, SURVEY N3) on the config's grid: Lele's "
                         "tenth-order compact LHS (1/20, 1/2, 1, 1/2, 1/20)")
    ap.add_argument("--no-phase-events", action="store_true",
                    help="measurement: the plan without CTRI_FLAG_TIMING (no per-phase events between "
                         "the kernels of a solve; comm_us and the live local-kernel time unavailable)")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every solve from the host instead of replaying one CUDA graph")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(cfg: str, p: int):
    import workloads
    dims, sd = workloads.config(cfg, p)
    names = {
        "cfg1": "64x8x8 fp64 cyclic B[1/3,1,1/3], solve index 0",
        "cfg2": "strong scaling: 8192x256x256 fp64 cyclic B[1/3,1,1/3], solve index 0",
        "cfg3": f"weak scaling: {256 * p}x256x256 (256^3 per GPU) fp64 cyclic, solve index 0",
        "cfg4_d1": "direction sweep: 256x8192x256, solve index 1",
        "cfg4_d2": "direction sweep: 256x256x8192, solve index 2 (contiguous)",
        "cfg5": "compact 6th-order first derivative 1024x512x512, stencil + solve, index 0",
    }
    return dims, sd, names[cfg]


# ------------------------------------------------------------------ clocks (nvidia-smi)
class ClockSampler:
    FIELDS = ("index,timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_indices):
        self.rows = []
        self.proc = None
        self.gpus = gpu_indices
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", ",".join(str(g) for g in self.gpus)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [c.strip() for c in line.split(",")]))

    def mark(self, which):
        if which == "start":
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        inside = [r for t, r in self.rows if self.t0 and self.t1 and self.t0 <= t <= self.t1]
        note = None
        if not inside:  # timed region shorter than the sampling period: nearest samples
            ts = [(abs(t - (self.t0 or t)), r) for t, r in self.rows]
            inside = [min(ts, key=lambda z: z[0])[1]]
            note = "timed region shorter than 50 ms sampling; nearest sample"
        sm = []
        mx = []
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in inside:
            try:
                sm.append(float(r[2]))
                mx.append(float(r[3]))
            except ValueError:
                pass
            for k, nm in enumerate(names):
                if len(r) > 6 + k and r[6 + k].lower() == "active":
                    reasons.add(nm)
        out = {"sm_mhz": statistics.median(sm) if sm else None,
               "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
               "samples": len(inside)}
        if note:
            out["note"] = note
        return out


# ------------------------------------------------------------------ CPU oracle baseline
def cpu_oracle_sample(cfg: str, budget_s: float = 10.0):
    """Time the oracle (as it stands) on a bounded sample of the workload: the full solve
    direction, a growing fraction of the batch columns, extrapolated to the full batch."""
    import numpy as np

    import oracle
    import workloads
    dims, sd, _ = workload(cfg, 1)
    n = dims[sd]
    other = [dims[k] for k in range(3) if k != sd]
    m_full = other[0] * other[1]
    m = min(m_full, 256)
    best = None
    while True:
        shape = [1, m, n] if sd == 2 else ([1, n, m] if sd == 1 else [n, 1, m])
        b = workloads.uniform(shape, 2)
        t0 = time.perf_counter()
        if cfg == "cfg5":
            oracle.deriv(b, sd)
        else:
            oracle.cyclic_solve(b, sd)
        dt = time.perf_counter() - t0
        best = (dt, m, tuple(shape))
        if dt >= budget_s / 3 or m >= m_full:
            break
        m = min(m_full, m * max(2, int(2 ** math.floor(math.log2(max(1.0, budget_s / 3 / max(dt, 1e-4)))))))
    dt, m, shape = best
    ms_full = dt * 1e3 * (m_full / m)
    out = {"value": ms_full, "unit": "ms", "cores": oracle.num_threads(), "kind": "oracle",
           "sample": f"{n} rows x {m} of {m_full} batch columns (shape {list(shape)}), "
                     f"{dt:.2f} s" + (f", extrapolated x{m_full / m:g} to the full batch" if m < m_full
                                      else " (the full workload)")}
    out.update(host_info())
    return out


def host_info():
    """The host cores the oracle runs on: nproc, the lscpu model and OpenMP threads used."""
    import oracle
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=5).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "omp_threads": oracle.num_threads()}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands (rank 0 only), on the same workload as the
    GPU arm: every step solves the FULL batch (all columns of the global grid) unless the
    requested steps would not fit in a few minutes, in which case each step solves a column
    sample and the line says so ("extrapolated": true).  Steps and warm-up are honoured."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    import oracle
    import workloads
    dims, sd, name = workload(args.config, world)
    n = dims[sd]
    m_full = int(np.prod(dims)) // n
    shape = [1, m_full, n] if sd == 2 else ([1, n, m_full] if sd == 1 else [n, 1, m_full])
    fn_of = (lambda a: oracle.deriv(a, sd)) if args.config == "cfg5" else (lambda a: oracle.cyclic_solve(a, sd))
    # probe one slice to size the run (<= 240 s for warm-up + timed steps)
    m_probe = min(m_full, 4096)
    pshape = list(shape)
    pshape[2 if sd != 2 else 1] = m_probe
    t0 = time.perf_counter()
    fn_of(workloads.uniform(pshape, 2))
    est_full = (time.perf_counter() - t0) * m_full / m_probe
    steps, warm = max(1, args.steps), max(0, args.warmup)
    budget = 240.0
    m = m_full
    if est_full * (steps + warm) > budget:
        m = max(256, int(m_full * budget / (est_full * (steps + warm))) // 256 * 256)
        m = min(m, m_full)
        shape[2 if sd != 2 else 1] = m
    b = workloads.uniform(shape, 2)
    for _ in range(warm):
        fn_of(b)
    t0 = time.perf_counter()
    for _ in range(steps):
        fn_of(b)
    dt = (time.perf_counter() - t0) / steps
    ms = dt * 1e3 * m_full / m
    extrap = m != m_full
    sample = (f"{n} rows x {m} of {m_full} batch columns per step" +
              (f", extrapolated x{m_full / m:g}" if extrap else " (the full workload every step)"))
    cpu = {"value": ms, "unit": "ms", "kind": "oracle", "sample": sample, "extrapolated": extrap}
    info = host_info()
    cpu["cores"] = info["omp_threads"]
    cpu.update(info)
    line = {"impl": "reference", "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world,
            "steps": steps, "warmup": warm, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong" if args.config != "cfg3" else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "global_dims": list(dims), "solve_dim": sd},
            "cpu_baseline": cpu,
            "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(cfg, p):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)
        return d.get(f"{cfg}_p{p}")  # dram read+write bytes per launch of the dominant kernel
    except Exception:
        return None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import workloads
    from paper_2101_02286_b200 import CTRI_FLAG_DERIV, CTRI_FLAG_TIMING, ctri
    from paper_2101_02286_b200 import dist as pdist

    rank, world, local = dist_env()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun --nproc-per-node N")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    p = world
    dims, sd, name = workload(args.config, p)
    if args.dims:
        dims = tuple(int(v) for v in args.dims.split(","))
        sd = args.sd
        name = f"custom {dims} solve index {sd}"
    deriv = args.config == "cfg5"
    # the timed region runs the plan a user runs: no per-phase events (CTRI_FLAG_TIMING puts an
    # event node between the kernels of a captured solve, which costs the programmatic launch
    # overlap: 14-20 us per multi-kernel solve, profiles/r2_events_ab.txt); a second plan with
    # the events measures the per-kernel times in its own timed pass (roofline, comm_us)
    flags = CTRI_FLAG_DERIV if deriv else 0
    if world > 1 and args.reduced == "fused":
        flags |= ctri.CTRI_FLAG_FUSED_REDUCED
    elif world > 1 and args.reduced == "allgather":
        flags |= ctri.CTRI_FLAG_ALLGATHER
    elif world > 1 and args.reduced == "nccl":
        flags |= ctri.CTRI_FLAG_NCCL_ROUNDS
    bands, coef = (1 / 3, 1.0, 1 / 3), None
    if deriv and args.scheme != "collocated":
        delta = 2 * math.pi / dims[sd]
        if args.scheme == "staggered_deriv":
            bands, coef = ctri.staggered_deriv_bands(), ctri.staggered_deriv_coef(delta)
        else:
            bands, coef = ctri.staggered_interp_bands(), ctri.staggered_interp_coef()
        name = f"{name.replace('compact 6th-order first derivative', args.scheme.replace('_', ' '))} (P:202-206)"
    if args.penta:
        if deriv:
            raise SystemExit("--penta applies to the solve configs (cfg1-cfg4)")
        bands = (1 / 20, 1 / 2, 1.0, 1 / 2, 1 / 20)
        name = f"pentadiagonal (Lele 10th-order LHS, r = 2): {name}"
    def make_plan(fl):
        if world > 1:
            return pdist.plan_from_process_group(dims, sd, bands, flags=fl)
        return ctri.Plan(dims, sd, 1, 0, bands=bands, flags=fl)

    plan = make_plan(flags)
    lshape = plan.local_shape
    b = workloads.device_uniform(lshape, 1000 * 2 + rank, dev)
    x = torch.empty_like(b)
    stream = torch.cuda.current_stream(dev)
    pts_local = b.numel()

    def solve_with(pl):
        def step():
            if coef is not None:
                pl.compact_apply(coef, b, x)
            elif deriv:
                pl.deriv(b, x)
            else:
                pl.solve(b, x)
        return step

    def prepare(step):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if args.no_graph:
            return step
        graph = torch.cuda.CUDAGraph()  # one solve captured as a CUDA graph, replayed per step
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()
        for _ in range(max(3, args.warmup)):
            graph.replay()
        torch.cuda.synchronize()
        prepare.graphs.append(graph)
        return graph.replay

    prepare.graphs = []
    step = solve_with(plan)
    timed_step = prepare(step)
    st0 = plan.stats()
    sampler = None
    if rank == 0:
        gpus = list(range(world)) if world > 1 else [local]
        sampler = ClockSampler(gpus)
        sampler.start()
        time.sleep(0.2)
    # timed region: K steps bracketed by barrier + synchronize, CUDA events on the solve stream
    local_us = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.mark("start")
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # one-launch solves (the virtual-partition chain): events around every step time the kernel
    # itself across the whole timed region (graph-replay overhead included)
    one_launch = st0["launches_per_solve"] == 1
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)] if one_launch else []
    e0.record(stream)
    for i in range(args.steps):
        if one_launch:
            kev[i][0].record(stream)
        timed_step()
        if one_launch:
            kev[i][1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    if sampler:
        sampler.mark("end")
    if world > 1:
        dist.barrier()
    ms_rank = e0.elapsed_time(e1) / args.steps
    ms = pdist.max_over_ranks(ms_rank, dev) if world > 1 else ms_rank
    # per-kernel / per-phase device times: a second plan with phase events (CTRI_FLAG_TIMING),
    # its own timed pass of the same steps (barrier + synchronize, graph replays back to back);
    # the plan's events around the local kernel in its last solve, and the mean over 50
    # isolated solves (each after a synchronize) beside it
    tplan = plan if args.no_phase_events else make_plan(flags | CTRI_FLAG_TIMING)
    tstep = solve_with(tplan)
    treplay = prepare(tstep)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        treplay()
    torch.cuda.synchronize()
    st = tplan.stats()
    for _ in range(min(50, args.steps)):
        tstep()
        local_us.append(tplan.stats()["t_local_us"])
    if sampler:
        sampler.stop()
    t_local_iso = statistics.mean(local_us)
    t_local_iso = pdist.max_over_ranks(t_local_iso, dev) if world > 1 else t_local_iso
    t_local = st["t_local_us"] if st["t_local_us"] > 0 else t_local_iso
    t_src = ("CUDA events (the plan's phase events) around the kernel in the last of a second timed "
             "pass of the same steps with a phase-event plan (graph replay)")
    if one_launch:
        t_local = 1e3 * statistics.mean(a.elapsed_time(b) for a, b in kev)
        t_src = "CUDA events around every timed step (the solve is one kernel launch)"
    t_local = pdist.max_over_ranks(t_local, dev) if world > 1 else t_local
    stage_us = [pdist.max_over_ranks(v, dev) if world > 1 else v for v in st["t_stage_us"]]
    yx = pdist.max_over_ranks(st["t_yexchange_us"], dev) if world > 1 else st["t_yexchange_us"]
    xx = pdist.max_over_ranks(st["t_xexchange_us"], dev) if world > 1 else st["t_xexchange_us"]
    back = pdist.max_over_ranks(st["t_backsub_us"], dev) if world > 1 else st["t_backsub_us"]
    p2p_k = pdist.max_over_ranks(st["t_reduced_kernel_us"], dev) if world > 1 else st["t_reduced_kernel_us"]
    win_k = pdist.max_over_ranks(st["t_window_us"], dev) if world > 1 else st["t_window_us"]

    # e2e through ctri_solve_host with pinned host buffers
    e2e = None
    if not args.no_e2e and not deriv:
        bh = b.cpu().pin_memory()
        xh = torch.empty_like(bh).pin_memory()
        plan.solve_host(bh, xh)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            plan.solve_host(bh, xh)
        f1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = f0.elapsed_time(f1) / args.e2e_steps
        e2e_ms = pdist.max_over_ranks(e2e_ms, dev) if world > 1 else e2e_ms
        nbytes = bh.numel() * 8
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "steps": args.e2e_steps,
               "path": "ctri_solve_host: pinned host -> HBM, solve, HBM -> pinned host; one "
                       "partition pipelines copies and solves over 16 column chunks"}
        del bh, xh

    if rank == 0:
        peak, peak_src = load_peaks()
        bytes_local = BYTES_PER_POINT * pts_local
        achieved = bytes_local / (t_local * 1e-6) / 1e9
        step_gbs = bytes_local / (ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": load_traffic(args.config, p),
                "kernel": ("k_tile<%d>%s (cluster %d)%s" % (st["rows_per_thread"],
                                                            " contiguous-axis" if st["local_kernel"] == 2 else "",
                                                            st["cluster_size"],
                                                            ", virtual-partition chain: (a1)-(a4) in one launch"
                                                            if (p == 1 and st["reduced_path"] == 3) else "")
                           if st["local_kernel"] in (1, 2) else
                           "k_penta_local (column-serial, 32 B/pt moved)" if st["local_kernel"] == 3
                           else "k_ptile (pentadiagonal on chip: register leaf + 2x2-block PCR, clusters)"
                           if st["local_kernel"] == 4
                           else "k_local_generic"),
                "algorithmic_bytes_per_launch": bytes_local, "launch_us": t_local,
                "launch_us_isolated": t_local_iso,
                "launch_us_source": t_src,
                "frac_nominal_8tbs": achieved / 8000.0,
                # context: the strided access pattern's own copy ceiling on B200 (6.0 TB/s with
                # every pipeline, profiles/r2_copy_ceiling_pattern.log; index-0/1 configs)
                "frac_of_pattern_copy_ceiling": achieved / 6000.0,
                "peak_source": peak_src}
        cpu = None if args.no_cpu_baseline else cpu_oracle_sample(args.config)
        launches = st["launches_per_solve"] * args.steps + (args.steps * 0)
        line = {"metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
                "scaling": "strong" if args.config != "cfg3" else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": name, "global_dims": list(dims), "solve_dim": sd,
                           "nparts": p, "local_dims": list(lshape),
                           "bands": list(bands), "cyclic": True,
                           "reduced": args.reduced if p > 1 else None,
                           "l2": "inputs larger than L2 (%.2f GB per array per GPU)" % (pts_local * 8 / 1e9),
                           "local_kernel": roof["kernel"],
                           "launch": "host launches" if args.no_graph else "one CUDA graph per solve"},
                "pct_hbm_roofline": 100.0 * step_gbs / peak,
                "pct_nominal_8tbs": 100.0 * step_gbs / 8000.0,  # north star: >= 60% of ~8 TB/s
                "step_gbs": step_gbs,
                "roofline": roof,
                "cpu_baseline": cpu,
                "e2e": e2e,
                "gpu_launches": launches,
                "comm_us": ({"reduced_phase_us": back,
                             "p2p_kernel_us": p2p_k, "window_kernel_us": win_k,
                             "per_round_median_us": {"y_exchange": st["t_p2p_y_us"],
                                                     "schedule_steps": st["t_p2p_step_us"],
                                                     "x_exchange": st["t_p2p_x_us"]},
                             "note": "device-initiated (a2)-(a4): LL P2P stores over NVLink "
                                     "(pairwise schedule, or one all-gather round), then the "
                                     "window back-substitution kernel; kernel times are CUDA "
                                     "events (max over ranks), rounds are medians over rank 0's "
                                     "CTAs of %globaltimer stamps; the y round includes waiting "
                                     "for the slowest peer's local solve"}
                            if st["reduced_path"] in (1, 2) else
                            {"fused_into_tile_kernel": True,
                             "note": "(a2)-(a4) inside the local-solve kernel: LL all-gather of the "
                                     "planes per tile, window rows finalised on chip one tile later"}
                            if st["reduced_path"] == 3 else
                            {"y_exchange": yx, "stages": stage_us, "x_exchange": xx,
                             "backsub_kernel": back}) if p > 1 else None,
                "clocks": sampler.summary() if sampler else None}
        print(json.dumps(line), flush=True)
    if tplan is not plan:
        tplan.close()
    plan.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
