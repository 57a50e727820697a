"""Shared test helpers: run the CUDA path through the C ABI on a global array and compare
with the oracle using the normwise-per-column metric of DESIGN.md reading R11."""
from __future__ import annotations

import numpy as np

import workloads

TOL_REL = 1e-12   # BASELINE.json north_star: max relative error <= 1e-12 (normwise per column)
TOL_RES = 1e-13   # residual ||Ax - b||_inf / ||b||_inf <= 1e-13


def columns(a: np.ndarray, sd: int) -> np.ndarray:
    return np.moveaxis(a, sd, 0).reshape(a.shape[sd], -1)


def rel_err(x: np.ndarray, ref: np.ndarray, sd: int) -> float:
    """max over columns of max_j |x - ref| / max_j |ref|."""
    xc, rc = columns(x, sd), columns(ref, sd)
    den = np.max(np.abs(rc), axis=0)
    den[den == 0] = 1.0
    return float(np.max(np.max(np.abs(xc - rc), axis=0) / den))


def residual(x: np.ndarray, b: np.ndarray, sd: int, bands=(1 / 3, 1.0, 1 / 3), cyclic=True) -> float:
    """max over columns of ||A x - b||_inf / ||b||_inf (band matvec)."""
    l, d, u = bands
    xc, bc = columns(x, sd), columns(b, sd)
    up = np.roll(xc, 1, axis=0)
    dn = np.roll(xc, -1, axis=0)
    if not cyclic:
        up[0] = 0
        dn[-1] = 0
    r = l * up + d * xc + u * dn - bc
    den = np.max(np.abs(bc), axis=0)
    den[den == 0] = 1.0
    return float(np.max(np.max(np.abs(r), axis=0) / den))


def gpu_solve(b_global: np.ndarray, sd: int, p: int = 1, bands=(1 / 3, 1.0, 1 / 3), cyclic=True,
              flags: int = 0, inplace: bool = False, return_stats: bool = False):
    """Solve through ctri_solve (p = 1) or the loopback group (p > 1) on cuda:0."""
    import torch

    from paper_2101_02286_b200 import ctri

    dev = torch.device("cuda:0")
    shape = b_global.shape
    slabs = [torch.from_numpy(workloads.slab(b_global, sd, p, r)).to(dev) for r in range(p)]
    xs = slabs if inplace else [torch.empty_like(s) for s in slabs]
    if p == 1:
        plan = ctri.Plan(shape, sd, 1, 0, bands, cyclic, None, flags)
        plan.solve(slabs[0], xs[0])
        torch.cuda.synchronize()
        st = plan.stats()
        plan.close()
    else:
        grp = ctri.LoopbackGroup(shape, sd, p, bands, cyclic, flags)
        grp.solve(slabs, xs)
        torch.cuda.synchronize()
        st = grp.stats(0)
        grp.close()
    x = workloads.assemble([t.cpu().numpy() for t in xs], sd)
    return (x, st) if return_stats else x
