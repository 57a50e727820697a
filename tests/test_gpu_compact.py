"""GPU parity of ctri_compact_apply (other bands and right-hand sides) against
the oracle: the staggered sixth-order derivative and interpolation of PAPER.md P:202-206 and a
general non-symmetric five-point stencil with non-symmetric bands, fused into the local-solve
tile kernel or as a separate stencil pass, on 1, 2, 4 and 8 partitions."""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import workloads
from helpers import rel_err

pytestmark = pytest.mark.gpu

CASES = [
    (1, (1024, 2, 16), 0, False), (2, (1024, 2, 16), 0, False), (4, (1024, 2, 16), 0, False),
    (1, (2048, 3, 16), 0, False),   # fused stencil across a 4-CTA cluster
    (1, (8192, 1, 16), 0, False),   # 16-CTA cluster, slab-edge halos from the wrap rows
    (2, (4, 1024, 32), 1, False),
    (8, (1024, 4, 16), 0, False),
    (3, (768, 2, 16), 0, False),    # detach / reattach reduced system with a halo
    (1, (1024, 2, 16), 0, True), (4, (1024, 2, 16), 0, True),  # unfused stencil + solve
    (2, (2, 3, 512), 2, False),     # contiguous axis
]


def _scheme(name, N):
    from paper_2101_02286_b200 import ctri
    h = 2 * math.pi / N
    if name == "sderiv":
        coef, ocoef, bands = ctri.staggered_deriv_coef(h), oracle.staggered_deriv_coef(h), ctri.staggered_deriv_bands()
    elif name == "sinterp":
        coef, ocoef, bands = ctri.staggered_interp_coef(), oracle.staggered_interp_coef(), ctri.staggered_interp_bands()
    else:  # a general five-point stencil with non-symmetric bands
        coef = ocoef = (0.3, -1.7, 0.25, 2.1, -0.6)
        bands = (0.2, 1.1, 0.4)
    # the binding's and the oracle's transcriptions of P:202-206 must agree exactly
    assert tuple(coef) == tuple(ocoef)
    return tuple(coef), tuple(bands)


def _run(p, shape, sd, generic, coef, bands, f):
    import torch

    from paper_2101_02286_b200 import CTRI_FLAG_DERIV, CTRI_FLAG_GENERIC_LOCAL, ctri
    flags = CTRI_FLAG_DERIV | (CTRI_FLAG_GENERIC_LOCAL if generic else 0)
    dev = torch.device("cuda:0")
    fs = [torch.from_numpy(workloads.slab(f, sd, p, r)).to(dev) for r in range(p)]
    ds = [torch.empty_like(t) for t in fs]
    if p == 1:
        plan = ctri.Plan(shape, sd, 1, 0, bands=bands, flags=flags)
        plan.compact_apply(coef, fs[0], ds[0])
        torch.cuda.synchronize()
        plan.close()
    else:
        g = ctri.LoopbackGroup(shape, sd, p, bands=bands, flags=flags)
        g.compact_apply(coef, fs, ds)
        torch.cuda.synchronize()
        g.close()
    return workloads.assemble([t.cpu().numpy() for t in ds], sd)


@pytest.mark.parametrize("scheme", ["sderiv", "sinterp", "general"])
@pytest.mark.parametrize("p,shape,sd,generic", CASES)
def test_compact_apply_matches_oracle(scheme, p, shape, sd, generic):
    N = shape[sd]
    coef, bands = _scheme(scheme, N)
    f = workloads.uniform(shape, 21) if scheme == "general" else workloads.cfg5_field(shape, sd, 5)
    out = _run(p, shape, sd, generic, coef, bands, f)
    ref = oracle.compact_apply(f, sd, coef, bands)
    assert rel_err(out, ref, sd) < 1e-12


@pytest.mark.parametrize("p", [1, 4])
def test_staggered_deriv_wavenumber_on_gpu(p):
    """GPU staggered derivative of sin at half nodes equals k'(k) cos at nodes (Fourier closed form)."""
    N, k = 1024, 37
    shape = (N, 2, 16)
    h = 2 * math.pi / N
    coef, bands = _scheme("sderiv", N)
    i = np.arange(N, dtype=np.int64)
    g = np.sin(math.pi * ((k * (2 * i + 1)) % (2 * N)) / N)
    f = np.broadcast_to(g.reshape(N, 1, 1), shape).copy()
    out = _run(p, shape, 0, False, coef, bands, f)
    kp = (2 * 63 / 62 * math.sin(k * h / 2) + 2 * 17 / 62 / 3 * math.sin(3 * k * h / 2)) / (
        1 + 2 * 9 / 62 * math.cos(k * h)) / h
    expect = kp * np.cos(2 * math.pi * ((k * i) % N) / N)
    assert np.max(np.abs(out - expect.reshape(N, 1, 1))) < 1e-12 * kp


def test_compact_apply_rejects_bad_coef():
    import torch

    from paper_2101_02286_b200 import CTRI_FLAG_DERIV, ctri
    shape = (64, 2, 16)
    plan = ctri.Plan(shape, 0, 1, 0, flags=CTRI_FLAG_DERIV)
    f = torch.zeros(shape, dtype=torch.float64, device="cuda:0")
    with pytest.raises(ctri.CtriError, match="INVALID_ARG"):
        plan.compact_apply((0, 1, float("nan"), 1, 0), f, torch.empty_like(f))
    plan.close()
