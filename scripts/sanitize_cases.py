"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Covers the tile kernel at cluster sizes G = 1, 2, 4 (cfg1-sized slabs), the fused stencil
variant, the loopback P2P reduced kernel (LL mailboxes) with the window pass, virtual
partitions on one GPU, and the pentadiagonal path.  Every case is checked against the oracle
so a sanitizer run that perturbs timing still has to produce the right answer.

usage: compute-sanitizer --tool racecheck python scripts/sanitize_cases.py [case ...]
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from helpers import gpu_solve, rel_err  # noqa: E402


def tile(shape):
    b = workloads.uniform(shape, 3)
    x, st = gpu_solve(b, 0, return_stats=True)
    e = rel_err(x, oracle.cyclic_solve(b, 0), 0)
    return f"tile {shape} G={st['cluster_size']} K={st['rows_per_thread']} vp={st['vparts']}", e


def loopback(p, shape=(1024, 2, 32)):
    b = workloads.uniform(shape, 4)
    x, st = gpu_solve(b, 0, p, return_stats=True)
    assert st["device_error"] == 0
    e = rel_err(x, oracle.cyclic_solve(b, 0), 0)
    return f"loopback p={p} {shape} path={st['reduced_path']}", e


def vparts(vp):
    os.environ["CTRI_VPARTS"] = str(vp)
    try:
        b = workloads.uniform((4096, 1, 32), 5)
        x, st = gpu_solve(b, 0, return_stats=True)
    finally:
        del os.environ["CTRI_VPARTS"]
    return f"virtual partitions vp={st['vparts']}", rel_err(x, oracle.cyclic_solve(b, 0), 0)


def deriv():
    import torch
    from paper_2101_02286_b200 import CTRI_FLAG_DERIV, ctri
    shape = (1024, 2, 32)
    f = workloads.cfg5_field(shape, 0, 5)
    ft = torch.from_numpy(f).cuda()
    dt = torch.empty_like(ft)
    with ctri.Plan(shape, 0, flags=CTRI_FLAG_DERIV) as plan:
        plan.deriv(ft, dt)
        torch.cuda.synchronize()
    return "fused stencil deriv", rel_err(dt.cpu().numpy(), oracle.deriv(f, 0), 0)


def contig():
    b = workloads.uniform((2, 16, 1024), 6)
    x = gpu_solve(b, 2)
    return "contiguous axis", rel_err(x, oracle.cyclic_solve(b, 2), 2)


def penta(p):
    import torch
    from paper_2101_02286_b200 import ctri
    bands = (0.05, 0.3, 1.0, 0.3, 0.05)
    shape = (256, 2, 32)
    b = workloads.uniform(shape, 7)
    dev = torch.device("cuda:0")
    slabs = [torch.from_numpy(workloads.slab(b, 0, p, r)).to(dev) for r in range(p)]
    xs = [torch.empty_like(s) for s in slabs]
    if p == 1:
        h = ctri.ctri_plan_create_penta(shape, 0, 1, 0, bands)
        ctri.ctri_solve(h, slabs[0], xs[0])
        torch.cuda.synchronize()
        ctri.ctri_plan_destroy(h)
    else:
        hs = ctri.ctri_plan_create_penta_loopback(shape, 0, p, bands)
        ctri.ctri_solve_loopback(hs, slabs, xs)
        torch.cuda.synchronize()
        for h in hs:
            ctri.ctri_plan_destroy(h)
    x = workloads.assemble([t.cpu().numpy() for t in xs], 0)
    return f"penta p={p}", rel_err(x, oracle.penta_solve(b, 0, bands), 0)


CASES = {
    "tile_g1": lambda: tile((256, 2, 32)),
    "tile_g2": lambda: tile((512, 1, 32)),
    "tile_g4": lambda: tile((1024, 1, 32)),
    "vparts": lambda: vparts(4),
    "loopback2": lambda: loopback(2),
    "loopback4": lambda: loopback(4),
    "deriv": deriv,
    "contig": contig,
    "penta1": lambda: penta(1),
    "penta2": lambda: penta(2),
}


def main(argv):
    names = argv or list(CASES)
    bad = 0
    for n in names:
        what, e = CASES[n]()
        ok = e < 1e-12
        bad += not ok
        print(f"[sanitize-case] {n}: {what}: rel err {e:.2e} {'ok' if ok else 'FAIL'}", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
