"""Observed normwise errors of the CUDA path vs the oracle for the near-singular bands
alpha = 0.45 and 0.499 (DESIGN reading R22): single GPU, loopback partitions, detach/reattach."""
import sys

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads  # noqa: E402
from helpers import gpu_solve, rel_err, residual  # noqa: E402

for a in (0.45, 0.499):
    bands = (a, 1.0, a)
    kappa = (1 + 2 * a) / (1 - 2 * a)
    worst, wres = 0.0, 0.0
    cases = [((512, 4, 32), 1, True), ((512, 4, 32), 1, False)]
    cases += [((64, 8, 8), p, True) for p in (2, 4, 8)] + [((1024, 4, 32), p, True) for p in (2, 4, 8)]
    cases += [((p * 16, 4, 16), p, True) for p in (3, 5, 6, 7, 11)]
    for shape, p, cyc in cases:
        b = workloads.uniform(shape, 6)
        x = gpu_solve(b, 0, p, bands, cyc)
        ref = oracle.cyclic_solve(b, 0, bands) if cyc else oracle.acyclic_solve(b, 0, bands)
        e, r = rel_err(x, ref, 0), residual(x, b, 0, bands, cyc)
        rr = residual(ref, b, 0, bands, cyc)
        worst, wres = max(worst, e), max(wres, r)
        print(f"alpha={a} shape={shape} p={p} cyclic={cyc}: rel_err={e:.3e} residual={r:.3e} oracle_residual={rr:.3e}")
    print(f"alpha={a}: kappa={kappa:.1f} kappa*u={kappa * 2**-53:.3e} worst rel_err={worst:.3e} worst residual={wres:.3e}")
