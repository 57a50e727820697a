"""The virtual-partition chain (tile-kernel LAYOUT 4) on one GPU: nparts == 1 with vp virtual
partitions whose reduced system (Eq. bi_hat, PCR, fold) and windowed
back-substitution (Eq. xi_app, reading R15) run inside the local-solve kernel.

Every case is compared element by element with the CPU oracle (Thomas + Sherman-Morrison, no
partitioning), and with the same plan built with CTRI_NO_VCHAIN=1 (k_reduced_local + k_window),
whose arithmetic differs only in rounding order.  Shapes cover: one column group (the
kernel's tail finalisation only), several groups per cluster, a ragged last column tile,
vp = 2 / 4 / 8, acyclic systems and non-symmetric bands.
"""
import numpy as np
import pytest

import oracle
import workloads
from helpers import TOL_REL, TOL_RES, rel_err, residual

pytestmark = pytest.mark.gpu

SYM = (1 / 3, 1.0, 1 / 3)
NONSYM = (0.2, 1.1, 0.4)


def _solve(b, bands, cyclic, monkeypatch, vchain=True, vp=None):
    import torch

    from paper_2101_02286_b200 import ctri
    if not vchain:
        monkeypatch.setenv("CTRI_NO_VCHAIN", "1")
    if vp is not None:
        monkeypatch.setenv("CTRI_VPARTS", str(vp))
    dev = torch.device("cuda:0")
    bt = torch.from_numpy(b).to(dev)
    xt = torch.empty_like(bt)
    plan = ctri.Plan(b.shape, 0, 1, 0, bands, cyclic)
    plan.solve(bt, xt)
    torch.cuda.synchronize()
    st = plan.stats()
    plan.close()
    return xt.cpu().numpy(), st


@pytest.mark.parametrize("shape,vp", [
    ((8192, 1, 32), 8),        # one column group: the tail finalises everything
    ((8192, 1, 40), 8),        # ragged: the second column tile holds 8 valid columns
    ((4096, 3, 96), 4),        # vp = 4, 9 column groups
    ((2048, 1, 64), 2),        # vp = 2 (knob), both partners of the single PCR stage coincide
    ((8192, 1, 32 * 150), 8),  # 150 groups: two or three per cluster, pipelined finalisation
])
@pytest.mark.parametrize("bands,cyclic", [(SYM, True), (SYM, False), (NONSYM, True)])
def test_vchain_matches_oracle(shape, vp, bands, cyclic, monkeypatch):
    b = workloads.uniform(shape, 17)
    x, st = _solve(b, bands, cyclic, monkeypatch, vp=vp)
    assert st["vparts"] == vp
    assert st["reduced_path"] == 3, "virtual-partition chain not taken"
    assert st["launches_per_solve"] == 1
    ref = oracle.cyclic_solve(b, 0, bands) if cyclic else oracle.acyclic_solve(b, 0, bands)
    assert rel_err(x, ref, 0) < TOL_REL
    assert residual(x, b, 0, bands, cyclic) < TOL_RES


@pytest.mark.parametrize("cyclic", [True, False])
def test_vchain_equals_separate_kernels(cyclic, monkeypatch):
    """Same plan, same input: the in-kernel chain and k_reduced_local + k_window agree to a few
    ulps (same method, only the rounding order of b^ differs)."""
    b = workloads.uniform((8192, 2, 64), 23)
    x1, st1 = _solve(b, SYM, cyclic, monkeypatch)
    x0, st0 = _solve(b, SYM, cyclic, monkeypatch, vchain=False)
    assert st1["reduced_path"] == 3 and st0["reduced_path"] == 0
    assert st0["launches_per_solve"] == 3
    assert np.max(np.abs(x1 - x0)) <= 1e-14 * np.max(np.abs(x0))


@pytest.mark.parametrize("r", [0, 1, 46, 47, 1023, 1024, 1025, 977, 2047, 8191])
def test_vchain_green_function(r, monkeypatch):
    """Unit impulse at and around the virtual partition edges (1024-row partitions): the
    solution is the periodic Green's function (closed form) -- window rows, row 0 (x~) and the
    rows just outside the window are all checked."""
    import math
    N, alpha = 8192, 1 / 3
    b = np.zeros((N, 1, 32))
    b[r] = 1.0
    x, st = _solve(b, (alpha, 1.0, alpha), True, monkeypatch)
    assert st["reduced_path"] == 3
    s = math.sqrt(1 - 4 * alpha * alpha)
    lam = (-1 + s) / (2 * alpha)
    d = (np.arange(N) - r) % N
    expect = (lam ** d + lam ** (N - d)) / (s * (1 - lam ** N))
    assert np.max(np.abs(x[:, 0, :] - expect[:, None])) < 1e-14


def test_vchain_repeated_solves(monkeypatch):
    """Back-to-back solves on one plan (the per-group barriers and buffers carry phase state
    only within a launch): 20 solves of alternating inputs, each against the oracle."""
    import torch

    from paper_2101_02286_b200 import ctri
    shape = (8192, 1, 32 * 75)
    bs = [workloads.uniform(shape, s) for s in (31, 32)]
    refs = [oracle.cyclic_solve(b, 0) for b in bs]
    dev = torch.device("cuda:0")
    plan = ctri.Plan(shape, 0)
    bt = [torch.from_numpy(b).to(dev) for b in bs]
    xt = torch.empty_like(bt[0])
    for k in range(20):
        plan.solve(bt[k % 2], xt)
        if k >= 18:
            torch.cuda.synchronize()
            assert rel_err(xt.cpu().numpy(), refs[k % 2], 0) < TOL_REL
    assert plan.stats()["reduced_path"] == 3
    plan.close()


@pytest.mark.parametrize("p,n,cyclic", [(2, 4096, True), (4, 2048, True), (3, 2048, True), (2, 4096, False),
                                        (2, 8192, True)])
@pytest.mark.parametrize("bands", [SYM, NONSYM])
def test_two_level_chain_loopback(p, n, cyclic, bands, monkeypatch):
    """nparts > 1 with virtual partitions chained in the tile kernel (two levels, opt-in): each rank's
    slab is solved as vp partitions whose internal interfaces are eliminated on chip
    (D_i^{-1} b_i of the whole slab), and the reduced system across the ranks has one row per
    rank (p = 3: detach / reattach).  Loopback on one GPU, every element vs the oracle."""
    from helpers import gpu_solve
    monkeypatch.setenv("CTRI_TWO_LEVEL", "1")
    b = workloads.uniform((p * n, 1, 64), 40 + p)
    x, st = gpu_solve(b, 0, p, bands, cyclic, return_stats=True)
    vp = min(8, n // 1024)
    assert st["vparts"] == vp and st["vchain"] == 1 and st["reduced_rows"] == p, st
    assert st["reduced_path"] == 1 and st["device_error"] == 0
    ref = oracle.cyclic_solve(b, 0, bands) if cyclic else oracle.acyclic_solve(b, 0, bands)
    assert rel_err(x, ref, 0) < TOL_REL
    assert residual(x, b, 0, bands, cyclic) < TOL_RES


@pytest.mark.parametrize("p", [2, 4])
def test_two_level_chain_cfg2_full_size(p, monkeypatch):
    """The BASELINE grid split into p loopback partitions of 4096 / 2048 rows (vp = 4 / 2
    chained on chip, p reduced rows): every one of the 65,536 columns vs the oracle."""
    import torch

    from paper_2101_02286_b200 import ctri
    from test_gpu_parity import _full_columns
    monkeypatch.setenv("CTRI_TWO_LEVEL", "1")
    dims = (8192, 256, 256)
    b = workloads.device_uniform(dims, 2, torch.device("cuda:0"))
    n = dims[0] // p
    bs = [b[r * n:(r + 1) * n].contiguous() for r in range(p)]
    xs = [torch.empty_like(t) for t in bs]
    g = ctri.LoopbackGroup(dims, 0, p)
    g.solve(bs, xs)
    torch.cuda.synchronize()
    st = g.stats(0)
    g.close()
    assert st["vchain"] == 1 and st["reduced_rows"] == p and st["device_error"] == 0
    err, m = _full_columns(b, torch.cat(xs, 0), 0)
    assert m == 65536 and err < TOL_REL, err
