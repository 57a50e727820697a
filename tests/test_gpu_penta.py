"""GPU parity of the pentadiagonal partition method (r = 2)
against the pentadiagonal oracle, through the C ABI: 1..8 partitions (loopback), cyclic and
acyclic, three band sets (incl. Lele's tenth-order LHS), all three solve directions, window and
full back-substitution, and the Fourier closed form."""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import workloads
from helpers import TOL_REL, rel_err

pytestmark = pytest.mark.gpu

BANDS = [(0.05, 0.3, 1.0, 0.3, 0.05), (-0.07, 0.21, 1.3, -0.33, 0.11), (1 / 20, 1 / 2, 1.0, 1 / 2, 1 / 20)]


def penta_gpu(b, sd, p, bands, cyclic=True, flags=0, inplace=False, return_stats=False):
    import torch

    from paper_2101_02286_b200 import ctri
    dev = torch.device("cuda:0")
    slabs = [torch.from_numpy(workloads.slab(b, sd, p, r)).to(dev) for r in range(p)]
    xs = slabs if inplace else [torch.empty_like(s) for s in slabs]
    if p == 1:
        plan = ctri.Plan(b.shape, sd, 1, 0, bands, cyclic, None, flags)
        plan.solve(slabs[0], xs[0])
        torch.cuda.synchronize()
        st = plan.stats()
        plan.close()
    else:
        g = ctri.LoopbackGroup(b.shape, sd, p, bands, cyclic, flags)
        g.solve(slabs, xs)
        torch.cuda.synchronize()
        st = g.stats(0)
        g.close()
    x = workloads.assemble([t.cpu().numpy() for t in xs], sd)
    return (x, st) if return_stats else x


def penta_residual(x, b, sd, bands, cyclic):
    xc = np.moveaxis(x, sd, 0)
    bc = np.moveaxis(b, sd, 0)
    r = -bc.copy()
    for off, v in zip((-2, -1, 0, 1, 2), bands):
        sh = np.roll(xc, -off, axis=0)
        if not cyclic:
            if off > 0:
                sh[-off:] = 0
            elif off < 0:
                sh[:-off] = 0
        r += v * sh
    return float(np.max(np.abs(r)) / np.max(np.abs(bc)))


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("cyclic", [True, False])
@pytest.mark.parametrize("bands", BANDS)
def test_penta_matches_oracle(p, cyclic, bands):
    shape = (12 * p, 3, 40)  # n = 12: reduced couplings far from negligible
    b = workloads.uniform(shape, 70 + p)
    x, st = penta_gpu(b, 0, p, bands, cyclic, return_stats=True)
    ref = oracle.penta_solve(b, 0, bands, cyclic)
    assert st["band_halfwidth"] == 2
    if p > 1:  # the pairwise block schedule; cyclic non-power-of-two p: block detach/reattach
        assert st["reduced_path"] == 1, st
        if cyclic and p & (p - 1):
            q = int(math.floor(math.log2(p)))
            assert st["detached_rows"] == p - 2 ** q and st["detach_stages"] == bin(p).count("1") - 1
    assert rel_err(x, ref, 0) < TOL_REL
    assert penta_residual(x, b, 0, bands, cyclic) < 1e-13


@pytest.mark.parametrize("p,shape,sd", [(1, (4096, 2, 64), 0), (2, (2048, 3, 40), 0), (4, (8, 1024, 32), 1),
                                        (2, (4, 8, 2048), 2), (8, (2048, 2, 33), 0), (1, (3, 5, 700), 2)])
@pytest.mark.parametrize("full", [False, True])
def test_penta_layouts_and_window(p, shape, sd, full):
    from paper_2101_02286_b200 import CTRI_FLAG_FULL_BACKSUB
    bands = BANDS[1]
    b = workloads.uniform(shape, 80 + p)
    x, st = penta_gpu(b, sd, p, bands, True, CTRI_FLAG_FULL_BACKSUB if full else 0, return_stats=True)
    assert rel_err(x, oracle.penta_solve(b, sd, bands, True), sd) < TOL_REL
    if not full and shape[sd] // p > 200:
        assert st["window_rows"] < shape[sd] // p // 2


def test_penta_inplace():
    b = workloads.uniform((1024, 2, 16), 90)
    x = penta_gpu(b, 0, 4, BANDS[0], inplace=True)
    assert rel_err(x, oracle.penta_solve(b, 0, BANDS[0], True), 0) < TOL_REL


@pytest.mark.parametrize("p", [1, 4])
def test_penta_fourier_closed_form(p):
    """b_j = cos(theta j) => x_j = Re(e^{i theta j} / lambda(theta)) (non-symmetric bands)."""
    e, l, d, u, f = BANDS[1]
    N, k = 2048, 301
    th = 2 * math.pi * k / N
    lam = d + l * np.exp(-1j * th) + u * np.exp(1j * th) + e * np.exp(-2j * th) + f * np.exp(2j * th)
    j = np.arange(N, dtype=np.int64)
    ph = 2 * math.pi * ((k * j) % N) / N
    b = np.broadcast_to(np.cos(ph).reshape(N, 1, 1), (N, 2, 16)).copy()
    x = penta_gpu(b, 0, p, BANDS[1])
    expect = np.real(np.exp(1j * ph) / lam).reshape(N, 1, 1)
    assert np.max(np.abs(x - expect)) < 1e-14


def test_penta_unsupported():
    from paper_2101_02286_b200 import CTRI_FLAG_DERIV, CTRI_FLAG_NCCL_ROUNDS, ctri
    with pytest.raises(ctri.CtriError, match="UNSUPPORTED"):
        ctri.LoopbackGroup((16 * 9, 2, 8), 0, 9, BANDS[0])
    with pytest.raises(ctri.CtriError, match="UNSUPPORTED"):
        ctri.Plan((64, 2, 8), 0, 1, 0, BANDS[0], True, None, CTRI_FLAG_DERIV)
    with pytest.raises(ctri.CtriError, match="UNSUPPORTED"):
        ctri.LoopbackGroup((64, 2, 8), 0, 2, BANDS[0], True, CTRI_FLAG_NCCL_ROUNDS)
    with pytest.raises(ctri.CtriError, match="PARTITION_TOO_SMALL"):
        ctri.LoopbackGroup((20, 2, 8), 0, 4, BANDS[0])


@pytest.mark.parametrize("p", [2, 4, 8])
def test_penta_pairwise_equals_allgather(p):
    """The two reduced-system solvers (2x2-block PCR, A^-1 all-gather) agree to rounding."""
    from paper_2101_02286_b200 import CTRI_FLAG_ALLGATHER
    b = workloads.uniform((16 * p, 2, 24), 120 + p)
    x1, s1 = penta_gpu(b, 0, p, BANDS[2], True, return_stats=True)
    x2, s2 = penta_gpu(b, 0, p, BANDS[2], True, CTRI_FLAG_ALLGATHER, return_stats=True)
    assert s1["reduced_path"] == 1 and s2["reduced_path"] == 2
    assert np.max(np.abs(x1 - x2)) < 1e-13 * np.max(np.abs(x2))



@pytest.mark.parametrize("r", [0, 1, 2, 15, 16, 17, 18, 63])
@pytest.mark.parametrize("cyclic", [True, False])
def test_penta_delta_at_partition_edges(r, cyclic):
    """A unit impulse on (and next to) the interface rows of a partition: the couplings through
    S, R, L~, U~ and the 2x2 reduced blocks are all exercised (p = 4, n = 16)."""
    N, p = 64, 4
    b = np.zeros((N, 1, 8))
    b[r] = 1.0
    for bands in BANDS:
        x = penta_gpu(b, 0, p, bands, cyclic)
        ref = oracle.penta_solve(b, 0, bands, cyclic)
        assert np.max(np.abs(x - ref)) < 1e-14 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("shape", [(256, 1, 64), (512, 2, 32), (1024, 1, 96), (8192, 1, 32), (4096, 2, 40)])
@pytest.mark.parametrize("cyclic", [True, False])
@pytest.mark.parametrize("bands", BANDS)
def test_penta_on_chip_matches_oracle(shape, cyclic, bands, monkeypatch):
    """The on-chip pentadiagonal local solve (ptile.cu): register leaf + 2x2-block PCR of the
    chunk heads; one partition of 256 / 512 / 1024 rows solved completely, longer slabs as
    n / 1024 partitions of one GPU (2x2-block PCR over them, then the window pass).  Every
    element vs the oracle, and vs the column-serial kernel of the same plan."""
    b = workloads.uniform(shape, 150 + shape[0] // 256)
    x, st = penta_gpu(b, 0, 1, bands, cyclic, return_stats=True)
    assert st["local_kernel"] == 4, st
    assert st["vparts"] == max(1, shape[0] // 1024)
    ref = oracle.penta_solve(b, 0, bands, cyclic)
    assert rel_err(x, ref, 0) < TOL_REL
    assert penta_residual(x, b, 0, bands, cyclic) < 1e-13
    monkeypatch.setenv("CTRI_PENTA_COLUMN_SERIAL", "1")
    xs, ss = penta_gpu(b, 0, 1, bands, cyclic, return_stats=True)
    assert ss["local_kernel"] == 3
    assert np.max(np.abs(x - xs)) < 1e-13 * np.max(np.abs(xs))


@pytest.mark.parametrize("r", [0, 1, 2, 31, 32, 33, 255, 256, 257, 1023, 1024, 1025, 2047])
def test_penta_on_chip_delta_at_chunk_and_partition_edges(r):
    """Unit impulses on and next to the chunk heads (every 32 rows), the CTA boundaries (256)
    and the on-GPU partition interfaces (1024) of the on-chip solve (p = 1, n = 2048: two
    partitions, clusters of 4)."""
    N = 2048
    b = np.zeros((N, 1, 32))
    b[r] = 1.0
    for bands in BANDS:
        for cyclic in (True, False):
            x, st = penta_gpu(b, 0, 1, bands, cyclic, return_stats=True)
            assert st["local_kernel"] == 4
            ref = oracle.penta_solve(b, 0, bands, cyclic)
            assert np.max(np.abs(x - ref)) < 1e-14 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("p", [1, 8])
def test_penta_cfg2_grid_full_size(p):
    """The pentadiagonal solve on the BASELINE grid (8192 x 256^2, Lele's tenth-order LHS) as
    bench.py --penta runs it (p = 1: 8 on-chip partitions; p = 8 loopback: 1024-row slabs on
    chip, reduced system over the P2P path): every column vs the oracle."""
    import torch

    from paper_2101_02286_b200 import ctri
    from test_gpu_parity import _full_columns
    bands = BANDS[2]
    dims = (8192, 256, 256)
    b = workloads.device_uniform(dims, 2, torch.device("cuda:0"))
    if p == 1:
        x = torch.empty_like(b)
        plan = ctri.Plan(dims, 0, 1, 0, bands)
        plan.solve(b, x)
        torch.cuda.synchronize()
        st = plan.stats()
        plan.close()
    else:
        n = dims[0] // p
        bs = [b[r * n:(r + 1) * n].contiguous() for r in range(p)]
        xs = [torch.empty_like(t) for t in bs]
        g = ctri.LoopbackGroup(dims, 0, p, bands)
        g.solve(bs, xs)
        torch.cuda.synchronize()
        st = g.stats(0)
        g.close()
        x = torch.cat(xs, 0)
    assert st["local_kernel"] == 4 and st["device_error"] == 0
    err, m = _full_columns(b, x, 0, fn=lambda a: oracle.penta_solve(a, 0, bands, True))
    assert m == 65536 and err < TOL_REL, err


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("cyclic", [True, False])
@pytest.mark.parametrize("vp", [1, 2])
def test_penta_on_chip_2048_row_slabs(p, cyclic, vp, monkeypatch):
    """Slabs of 2048 rows per rank (the cfg2 grid at 4 GPUs): vp = 1, the on-chip solve with
    clusters of 8 (64 chunk heads per column, 2x2-block PCR through shared memory); vp = 2, two
    1024-row partitions per rank as virtual rows of the reduced system; then the reduced system
    over the P2P path and the window pass; vs the oracle."""
    monkeypatch.setenv("CTRI_VPARTS", str(vp))
    b = workloads.uniform((2048 * p, 1, 64), 170 + p)
    for bands in BANDS:
        x, st = penta_gpu(b, 0, p, bands, cyclic, return_stats=True)
        assert st["local_kernel"] == 4 and st["device_error"] == 0
        assert st["vparts"] == vp and st["reduced_rows"] == p * vp
        ref = oracle.penta_solve(b, 0, bands, cyclic)
        assert rel_err(x, ref, 0) < TOL_REL
        assert penta_residual(x, b, 0, bands, cyclic) < 1e-13


@pytest.mark.parametrize("p,n", [(2, 4096), (3, 2048), (3, 4096), (4, 2048), (2, 2048)])
@pytest.mark.parametrize("cyclic", [True, False])
def test_penta_virtual_rows_multi_partition(p, n, cyclic):
    """nparts > 1 with slabs longer than 1024 rows: every slab solved on chip as n / 1024
    partitions, the reduced 2x2-block system over nparts * vp block rows on the P2P path
    (pairwise block PCR; block detach / reattach when the count is not a power of two),
    then the window pass; vs the oracle for the three band sets."""
    vp = n // 1024
    b = workloads.uniform((n * p, 1, 32), 190 + p + n // 1024)
    for bands in BANDS:
        x, st = penta_gpu(b, 0, p, bands, cyclic, return_stats=True)
        assert st["local_kernel"] == 4 and st["device_error"] == 0
        assert st["vparts"] == vp and st["reduced_rows"] == p * vp, st
        pr = p * vp
        if cyclic and pr & (pr - 1):
            assert st["detached_rows"] == pr - 2 ** int(math.floor(math.log2(pr)))
        ref = oracle.penta_solve(b, 0, bands, cyclic)
        assert rel_err(x, ref, 0) < TOL_REL
        assert penta_residual(x, b, 0, bands, cyclic) < 1e-13


@pytest.mark.parametrize("r", [0, 1, 2, 1022, 1023, 1024, 1025, 2047, 2048, 2049, 3071, 3072, 3073, 4095])
def test_penta_virtual_rows_delta_at_edges(r):
    """Unit impulses on and next to the virtual-row interfaces (every 1024 rows) and the rank
    interfaces (2048) of p = 2 slabs of 2048 rows (4 block rows in the reduced system)."""
    N, p = 4096, 2
    b = np.zeros((N, 1, 32))
    b[r] = 1.0
    for bands in BANDS:
        for cyclic in (True, False):
            x, st = penta_gpu(b, 0, p, bands, cyclic, return_stats=True)
            assert st["vparts"] == 2 and st["reduced_rows"] == 4
            ref = oracle.penta_solve(b, 0, bands, cyclic)
            assert np.max(np.abs(x - ref)) < 1e-14 * max(1.0, np.max(np.abs(ref)))


def test_misaligned_slabs_rejected():
    """The tile kernels stream b by TMA and the window passes move 16-byte column pairs: a slab
    pointer that is only 8-byte aligned is refused with INVALID_ARG (tridiagonal and
    pentadiagonal plans), never run."""
    import torch

    from paper_2101_02286_b200 import ctri
    dims = (2048, 1, 32)
    n = 2048 * 32
    buf = torch.zeros(n + 1, dtype=torch.float64, device="cuda:0")
    ok = torch.zeros(n, dtype=torch.float64, device="cuda:0")
    for bands in [(1 / 3, 1.0, 1 / 3), BANDS[2]]:
        plan = ctri.Plan(dims, 0, 1, 0, bands)
        with pytest.raises(ctri.CtriError, match="INVALID_ARG"):
            plan.solve(buf[1:], ok)
        with pytest.raises(ctri.CtriError, match="INVALID_ARG"):
            plan.solve(ok, buf[1:])
        plan.solve(ok, buf[:n])  # (aligned: runs)
        plan.close()


@pytest.mark.parametrize("n,vp", [(6144, 6), (5120, 5), (3072, 6), (7168, 7)])
@pytest.mark.parametrize("cyclic", [True, False])
def test_penta_one_gpu_non_power_of_two_partitions(n, vp, cyclic):
    """One GPU, n not a power-of-two multiple of 1024: vp on-chip partitions of a power-of-two
    length; the cyclic 2x2-block reduced system (vp not a power of two) by its plan-time
    inverse, the acyclic one by block PCR; vs the oracle for the three band sets."""
    b = workloads.uniform((n, 1, 32), 400 + vp)
    for bands in BANDS:
        x, st = penta_gpu(b, 0, 1, bands, cyclic, return_stats=True)
        assert st["local_kernel"] == 4 and st["vparts"] == vp, st
        ref = oracle.penta_solve(b, 0, bands, cyclic)
        assert rel_err(x, ref, 0) < TOL_REL
        assert penta_residual(x, b, 0, bands, cyclic) < 1e-13
