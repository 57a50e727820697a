"""GPU parity of the all-gather reduced solve (CTRI_FLAG_ALLGATHER): one exchange
round of 2 planes per rank and plan-time rows of A^{-1} instead of the 2 + log2 p pairwise
rounds.  Same oracle, same bar; partition edges pinned by the periodic Green's function."""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import workloads
from helpers import TOL_REL, TOL_RES, gpu_solve, rel_err, residual

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("cyclic", [True, False])
@pytest.mark.parametrize("bands", [(1 / 3, 1.0, 1 / 3), (0.45, 1.0, 0.45), (0.2, 1.1, 0.4)])
def test_allgather_matches_oracle(p, cyclic, bands):
    from paper_2101_02286_b200 import CTRI_FLAG_ALLGATHER
    shape = (16 * p, 3, 40)  # n = 16: reduced couplings far from negligible
    b = workloads.uniform(shape, 30 + p)
    x, st = gpu_solve(b, 0, p, bands, cyclic, flags=CTRI_FLAG_ALLGATHER, return_stats=True)
    ref = oracle.cyclic_solve(b, 0, bands) if cyclic else oracle.acyclic_solve(b, 0, bands)
    assert st["reduced_path"] == 2 and st["comm_rounds"] == 1
    assert rel_err(x, ref, 0) < TOL_REL
    assert residual(x, b, 0, bands, cyclic) < TOL_RES


@pytest.mark.parametrize("p,shape,sd", [(2, (2048, 4, 64), 0), (4, (8, 1024, 32), 1), (8, (4, 8, 2048), 2),
                                        (4, (1024, 2, 200), 0)])
def test_allgather_layouts(p, shape, sd):
    from paper_2101_02286_b200 import CTRI_FLAG_ALLGATHER
    b = workloads.uniform(shape, 40 + p)
    x = gpu_solve(b, sd, p, flags=CTRI_FLAG_ALLGATHER)
    assert rel_err(x, oracle.cyclic_solve(b, sd), sd) < TOL_REL


@pytest.mark.parametrize("r", [0, 15, 16, 17, 63])
def test_allgather_green_function_at_partition_edges(r):
    from paper_2101_02286_b200 import CTRI_FLAG_ALLGATHER
    N, p, alpha = 64, 4, 0.45
    b = np.zeros((N, 1, 8))
    b[r] = 1.0
    x = gpu_solve(b, 0, p, (alpha, 1.0, alpha), flags=CTRI_FLAG_ALLGATHER)[:, 0, 0]
    s = math.sqrt(1 - 4 * alpha * alpha)
    lam = (-1 + s) / (2 * alpha)
    d = (np.arange(N) - r) % N
    expect = (lam ** d + lam ** (N - d)) / (s * (1 - lam ** N))
    assert np.max(np.abs(x - expect)) < 1e-13


def test_allgather_deriv_and_repeat():
    """Derivative through the all-gather path, solved twice (mailbox epochs alternate)."""
    import torch

    from paper_2101_02286_b200 import CTRI_FLAG_ALLGATHER, CTRI_FLAG_DERIV, ctri
    p, shape = 4, (1024, 2, 16)
    f = workloads.cfg5_field(shape, 0, 5)
    ref = oracle.deriv(f, 0)
    dev = torch.device("cuda:0")
    fs = [torch.from_numpy(workloads.slab(f, 0, p, r)).to(dev) for r in range(p)]
    ds = [torch.empty_like(t) for t in fs]
    g = ctri.LoopbackGroup(shape, 0, p, flags=CTRI_FLAG_DERIV | CTRI_FLAG_ALLGATHER)
    for _ in range(3):
        g.deriv(fs, ds)
        torch.cuda.synchronize()
        assert rel_err(workloads.assemble([t.cpu().numpy() for t in ds], 0), ref, 0) < TOL_REL
    g.close()


def test_allgather_unsupported():
    from paper_2101_02286_b200 import CTRI_FLAG_ALLGATHER, CTRI_FLAG_NCCL_ROUNDS, ctri
    with pytest.raises(ctri.CtriError, match="UNSUPPORTED"):
        ctri.LoopbackGroup((16 * 9, 2, 8), 0, 9, flags=CTRI_FLAG_ALLGATHER)
    with pytest.raises(ctri.CtriError, match="UNSUPPORTED"):
        ctri.LoopbackGroup((64, 2, 8), 0, 2, flags=CTRI_FLAG_ALLGATHER | CTRI_FLAG_NCCL_ROUNDS)
