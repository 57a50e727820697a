"""Host pre-factorisation tables against dense linear algebra.

The plan's fp64 tables are host C++ (paper_2101_02286_b200/csrc/factor.cpp);
here they are checked without a GPU against dense inverses, the dense Schur
complement of the permuted system (block-LU reading), the paper's
stage counts and the golden PCR step of tests/golden/pcr_reduced_p4.txt.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import paper_2101_02286_b200 as pk

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
BANDS = [(1 / 3, 1.0, 1 / 3), (0.2, 1.1, 0.4), (-0.3, 1.0, 0.25), (0.45, 1.0, 0.45)]


def dense_acyclic(N, bands):
    l, d, u = bands
    return np.diag(np.full(N, d)) + np.diag(np.full(N - 1, l), -1) + np.diag(np.full(N - 1, u), 1)


def dense_cyclic(N, bands):
    l, d, u = bands
    A = np.zeros((N, N))
    for i in range(N):
        A[i, i] += d
        A[i, (i - 1) % N] += l
        A[i, (i + 1) % N] += u
    return A


@pytest.mark.parametrize("bands", BANDS)
@pytest.mark.parametrize("n", [3, 4, 8, 33, 256])
def test_S_R_vs_dense_inverse(bands, n):
    """Eqs. Si, Ri: D S = L (= l e_0), D R = U (= u e_last) with D the (n-1)-row interior block."""
    S, R, hat, w = pk.ctri_factor_query(n, bands)
    l, d, u = bands
    Dinv = np.linalg.inv(dense_acyclic(n - 1, bands))
    assert np.max(np.abs(S - l * Dinv[:, 0])) < 1e-15
    assert np.max(np.abs(R - u * Dinv[:, -1])) < 1e-15
    # Eqs. Li_hat, Di_hat, Ui_hat
    assert hat[0] == pytest.approx(-l * S[-1], abs=1e-18)
    assert hat[1] == pytest.approx(d - l * R[-1] - u * S[0], abs=1e-15)
    assert hat[2] == pytest.approx(-u * R[0], abs=1e-18)


def test_symmetric_limits_and_persymmetry():
    a = 1 / 3
    S, R, hat, w = pk.ctri_factor_query(8192)
    lam = (-1 + math.sqrt(1 - 4 * a * a)) / (2 * a)
    assert S[0] == pytest.approx(abs(lam), abs=1e-16)  # S[0] -> |lambda|
    assert hat[1] == pytest.approx(math.sqrt(1 - 4 * a * a), abs=1e-15)  # D^ -> sqrt(5)/3
    assert np.max(np.abs(S - R[::-1])) < 1e-16  # persymmetry S[k] = R[N-1-k]
    assert hat[0] == 0.0 and hat[2] == 0.0  # S underflows to exactly 0 for N_i >~ 774
    for n, expect in ((8, -3.38e-4), (32, -3.1e-14), (256, -7.4e-108)):
        _, _, h, _ = pk.ctri_factor_query(n)
        assert h[0] == pytest.approx(expect, rel=0.02), (n, h[0])


def test_window():
    """W = rows per end with |S| or |R| > 2^-64 (R15): 46 at alpha = 1/3."""
    for n in (256, 1024, 8192):
        assert pk.ctri_factor_query(n)[3] == 46
    S, R, _, w = pk.ctri_factor_query(1024)
    tau = 2.0 ** -64
    inner = np.r_[np.zeros(w, bool), np.ones(1023 - 2 * w, bool), np.zeros(w, bool)]
    assert np.all(np.abs(S[inner]) <= tau) and np.all(np.abs(R[inner]) <= tau)
    assert abs(S[w - 1]) > tau
    # alpha -> 1/2 widens the window to every row at small n
    assert pk.ctri_factor_query(64, (0.499, 1, 0.499))[3] == 63


def schur_reduced(N, p, bands, cyclic=True):
    """Dense Schur complement of the interface unknowns (rows i*n) -- block-LU reading P:254."""
    A = dense_cyclic(N, bands) if cyclic else dense_acyclic(N, bands)
    n = N // p
    I = [i * n for i in range(p)]
    J = [r for r in range(N) if r % n]
    AII = A[np.ix_(I, I)]
    AIJ = A[np.ix_(I, J)]
    AJI = A[np.ix_(J, I)]
    AJJ = A[np.ix_(J, J)]
    return AII - AIJ @ np.linalg.solve(AJJ, AJI)


@pytest.mark.parametrize("bands", BANDS)
@pytest.mark.parametrize("p,n", [(2, 8), (4, 8), (8, 4), (4, 33)])
def test_reduced_system_is_schur_complement(bands, p, n):
    """Eq. sub-system: the reduced system equals the dense Schur complement, cyclic wrap included."""
    _, _, (Lh, Dh, Uh), _ = pk.ctri_factor_query(n, bands)
    Ah = np.zeros((p, p))
    for i in range(p):
        Ah[i, i] += Dh
        Ah[i, (i - 1) % p] += Lh
        Ah[i, (i + 1) % p] += Uh
    Sc = schur_reduced(n * p, p, bands)
    assert np.max(np.abs(Ah - Sc)) < 1e-14


def apply_pcr(alpha, gamma, inv, b, cyclic=True):
    """Apply the PCR multipliers to a RHS (P:84 step structure), for checking the tables."""
    q, P = alpha.shape if alpha.size else (0, len(inv))
    b = np.array(b, dtype=np.float64)
    for k in range(q):
        s = 1 << k
        nb = b.copy()
        for c in range(P):
            lm, lp = c - s, c + s
            vm = b[lm % P] if (cyclic or lm >= 0) else 0.0
            vp = b[lp % P] if (cyclic or lp < P) else 0.0
            nb[c] = b[c] - alpha[k, c] * vm - gamma[k, c] * vp
        b = nb
    return b * inv


@pytest.mark.parametrize("P", [1, 2, 4, 8, 16, 64])
def test_cyclic_pcr_tables_vs_dense(P):
    rng = np.random.default_rng(P)
    L = rng.uniform(-0.4, 0.4, P)
    U = rng.uniform(-0.4, 0.4, P)
    D = rng.uniform(1.0, 1.3, P)
    a, g, inv = pk.ctri_pcr_coefficients(L, D, U, cyclic=True)
    assert a.shape[0] == int(math.log2(P))  # floor(log2 p) stages
    A = np.zeros((P, P))
    for c in range(P):
        A[c, c] += D[c]
        A[c, (c - 1) % P] += L[c]
        A[c, (c + 1) % P] += U[c]
    for _ in range(3):
        b = rng.uniform(-1, 1, P)
        x = apply_pcr(a, g, inv, b, True)
        assert np.max(np.abs(x - np.linalg.solve(A, b))) < 1e-14


@pytest.mark.parametrize("P", [1, 2, 3, 5, 7, 8, 13])
def test_acyclic_pcr_tables_vs_dense(P):
    rng = np.random.default_rng(100 + P)
    L = rng.uniform(-0.4, 0.4, P)
    U = rng.uniform(-0.4, 0.4, P)
    D = rng.uniform(1.0, 1.3, P)
    a, g, inv = pk.ctri_pcr_coefficients(L, D, U, cyclic=False)
    assert a.shape[0] == (math.ceil(math.log2(P)) if P > 1 else 0)  # ceil(log2 p)
    A = np.diag(D) + np.diag(L[1:], -1) + np.diag(U[:-1], 1)
    b = rng.uniform(-1, 1, P)
    assert np.max(np.abs(apply_pcr(a, g, inv, b, False) - np.linalg.solve(A, b))) < 1e-14


def test_golden_pcr_step_p4():
    """tests/golden/pcr_reduced_p4.txt (fold reading R3)."""
    gold = {}
    for line in open(os.path.join(GOLDEN, "pcr_reduced_p4.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, num, den = line.split()
        gold[k] = Fraction(int(num), int(den))
    a, g, inv = pk.ctri_pcr_coefficients([1 / 3] * 4, [1.0] * 4, [1 / 3] * 4, cyclic=True)
    assert a.shape == (2, 4)
    # stage 0: alpha = gamma = 1/3 -> new diagonal 1 - 2/9 = 7/9, new off-diagonal -1/9
    assert np.allclose(a[0], 1 / 3) and np.allclose(g[0], 1 / 3)
    d0 = 1 - a[0, 0] / 3 - g[0, 0] / 3
    off0 = -a[0, 0] / 3
    assert d0 == pytest.approx(float(gold["stage0_diag"]), abs=1e-15)
    assert off0 == pytest.approx(float(gold["stage0_off"]), abs=1e-15)
    # stage 1: alpha = off0 / d0 = -1/7; fold gives 5/7
    assert a[1, 0] == pytest.approx(float(gold["stage0_off"] / gold["stage0_diag"]), abs=1e-15)
    assert 1 / inv[0] == pytest.approx(float(gold["fold_diag"]), abs=1e-15)
    x = apply_pcr(a, g, inv, np.ones(4))
    assert np.allclose(x, float(gold["x"]), rtol=0, atol=1e-15)


# ---------------------------------------------------------------- reduced-system schedule (N2)
def run_schedule(kinds, w, src, c, b):
    """Execute the step schedule on a RHS (synchronous semantics, include/ctri.h)."""
    v = np.array(b, dtype=np.float64)
    for s in range(len(kinds)):
        nv = w[s] * v
        for k in range(2):
            idx = src[s, :, k]
            term = np.where(idx >= 0, v[np.maximum(idx, 0)], 0.0)
            nv = nv - c[s, :, k] * term
        v = nv
    return v


def dense_band(L, D, U, cyclic):
    P = len(D)
    A = np.zeros((P, P))
    for i in range(P):
        A[i, i] += D[i]
        if cyclic or i > 0:
            A[i, (i - 1) % P] += L[i]
        if cyclic or i < P - 1:
            A[i, (i + 1) % P] += U[i]
    return A


@pytest.mark.parametrize("P", list(range(1, 17)) + [23, 31, 33])
@pytest.mark.parametrize("cyclic", [True, False])
def test_reduced_schedule_vs_dense(P, cyclic):
    rng = np.random.default_rng(1000 + P)
    L = rng.uniform(-0.4, 0.4, P)
    U = rng.uniform(-0.4, 0.4, P)
    D = rng.uniform(1.0, 1.3, P)
    kinds, w, src, c, cnt = pk.ctri_reduced_schedule(L, D, U, cyclic=cyclic, max_steps=64)
    A = dense_band(L, D, U, cyclic)
    for _ in range(3):
        b = rng.uniform(-1, 1, P)
        assert np.max(np.abs(run_schedule(kinds, w, src, c, b) - np.linalg.solve(A, b))) < 1e-14
    if cyclic:  # stage counts
        q = int(math.floor(math.log2(P)))
        assert cnt["pcr_stages"] == q
        assert cnt["detached_rows"] == P - 2 ** q
        assert cnt["detach_stages"] == sum((P >> n) & 1 for n in range(q + 1)) - 1
    else:
        assert cnt["pcr_stages"] == (math.ceil(math.log2(P)) if P > 1 else 0)
        assert cnt["detach_stages"] == 0


def test_reduced_schedule_worked_example_11():
    """The paper's 11x11 walkthrough (tests/golden/detach_11x11.txt)."""
    P = 11
    kinds, w, src, c, cnt = pk.ctri_reduced_schedule([1 / 3] * P, [1.0] * P, [1 / 3] * P)
    names = {0: "detach", 1: "pcr", 2: "fold", 3: "reattach"}
    gold = {}
    for line in open(os.path.join(GOLDEN, "detach_11x11.txt")):
        if line.startswith("#") or not line.strip():
            continue
        f = line.split()
        gold.setdefault(int(f[0]), []).append((f[1], [int(x) for x in f[2:]]))
    assert len(kinds) == len(gold)
    for s, entries in gold.items():
        assert names[int(kinds[s])] == entries[0][0]
        if entries[0][0] == "detach":
            got = set()
            for r in range(P):  # rows that eliminate a detached row this step
                if src[s, r, 0] >= 0:
                    got.add((int(src[s, r, 0]) + 1, r + 1))
            want = set()
            for _, (z, y, a) in entries:
                want |= {(z, y), (z, a)}
            assert got == want, (s, got, want)
        if entries[0][0] == "reattach":
            got = {(r + 1, int(src[s, r, 0]) + 1, int(src[s, r, 1]) + 1) for r in range(P)
                   if src[s, r, 0] >= 0}
            assert got == {tuple(e[1]) for e in entries}, (s, got)
    assert cnt == {"pcr_stages": 3, "detach_stages": 2, "detached_rows": 3}
    # and it solves the benchmark reduced system (b = 1 -> x~ = 1 / (L+D+U) row sums)
    b = np.ones(P)
    A = dense_band([1 / 3] * P, [1.0] * P, [1 / 3] * P, True)
    assert np.allclose(run_schedule(kinds, w, src, c, b), np.linalg.solve(A, b), rtol=0, atol=1e-15)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 7, 8])
@pytest.mark.parametrize("cyclic", [True, False])
def test_reduced_inverse_vs_dense(P, cyclic):
    """All-gather table: ctri_reduced_inverse is the dense inverse of A^."""
    rng = np.random.default_rng(2000 + P)
    L = rng.uniform(-0.4, 0.4, P)
    U = rng.uniform(-0.4, 0.4, P)
    D = rng.uniform(1.0, 1.3, P)
    inv = pk.ctri_reduced_inverse(L, D, U, cyclic=cyclic)
    A = dense_band(L, D, U, cyclic)
    assert np.max(np.abs(inv @ A - np.eye(P))) < 1e-14
    assert np.max(np.abs(inv - np.linalg.inv(A))) < 1e-14


def test_reduced_inverse_singular():
    with pytest.raises(pk.CtriError, match="SINGULAR"):
        pk.ctri_reduced_inverse([0.5, 0.5], [1.0, 1.0], [0.5, 0.5], cyclic=True)  # [[1, 1], [1, 1]]


# ---- pentadiagonal (r = 2) partition tables ----
PENTA_BANDS = [(0.05, 0.3, 1.0, 0.3, 0.05), (-0.07, 0.21, 1.3, -0.33, 0.11), (1 / 20, 1 / 2, 1.0, 1 / 2, 1 / 20)]


def _dense_penta(N, bands, cyclic):
    A = np.zeros((N, N))
    for i in range(N):
        for off, v in zip((-2, -1, 0, 1, 2), bands):
            j = i + off
            if 0 <= j < N:
                A[i, j] += v
            elif cyclic:
                A[i, j % N] += v
    return A


@pytest.mark.parametrize("bands", PENTA_BANDS)
@pytest.mark.parametrize("n", [6, 7, 12, 40])
def test_penta_S_R_vs_dense(bands, n):
    """S = D^{-1} L, R = D^{-1} U with the interior block and couplings of P:212 (r = 2)."""
    e, l, d, u, f = bands
    N = n - 2
    t = pk.ctri_penta_factor_query(n, bands)
    D = _dense_penta(N, bands, False)
    L = np.zeros((N, 2))
    L[0, 0], L[0, 1], L[1, 1] = e, l, e
    U = np.zeros((N, 2))
    U[N - 2, 0], U[N - 1, 0], U[N - 1, 1] = f, u, f
    assert np.max(np.abs(t["S"] - np.linalg.solve(D, L))) < 1e-14
    assert np.max(np.abs(t["R"] - np.linalg.solve(D, U))) < 1e-14


@pytest.mark.parametrize("bands", PENTA_BANDS)
@pytest.mark.parametrize("p,n,cyclic", [(3, 10, True), (4, 8, True), (3, 12, False), (2, 9, True), (1, 11, True)])
def test_penta_reduced_blocks_are_the_schur_complement(bands, p, n, cyclic):
    """Eliminating every interior row of the assembled matrix leaves exactly the 2x2-block
    tridiagonal reduced matrix [L^, D^, U^] (D^ of the first partition without L~R when
    acyclic) -- the block-LU statement of P:254 with r = 2."""
    Ntot = p * n
    A = _dense_penta(Ntot, bands, cyclic)
    iface = [i * n + k for i in range(p) for k in (0, 1)]
    inter = [i for i in range(Ntot) if i not in iface]
    Aii = A[np.ix_(iface, iface)]
    Aij = A[np.ix_(iface, inter)]
    Aji = A[np.ix_(inter, iface)]
    Ajj = A[np.ix_(inter, inter)]
    schur = Aii - Aij @ np.linalg.solve(Ajj, Aji)
    t = pk.ctri_penta_factor_query(n, bands)
    expect = np.zeros((2 * p, 2 * p))
    for i in range(p):
        expect[2 * i:2 * i + 2, 2 * i:2 * i + 2] += t["Dh"] if (cyclic or i > 0) else t["Dh_first"]
        if cyclic or i > 0:
            j = (i - 1) % p
            expect[2 * i:2 * i + 2, 2 * j:2 * j + 2] += t["Lh"]
        if cyclic or i < p - 1:
            j = (i + 1) % p
            expect[2 * i:2 * i + 2, 2 * j:2 * j + 2] += t["Uh"]
    assert np.max(np.abs(schur - expect)) < 1e-13


@pytest.mark.parametrize("bands", PENTA_BANDS)
def test_penta_window(bands):
    """Outside the window every |S|, |R| entry is <= 2^-64 (reading R15 with r = 2)."""
    n = 2048
    t = pk.ctri_penta_factor_query(n, bands)
    W, N = t["window"], n - 2
    assert 0 < W < N // 2
    mid = slice(W, N - W)
    assert np.max(np.abs(t["S"][mid])) <= 2.0 ** -64
    assert np.max(np.abs(t["R"][mid])) <= 2.0 ** -64
    assert max(np.max(np.abs(t["S"][W - 1])), np.max(np.abs(t["R"][N - W]))) > 2.0 ** -64


def test_penta_singular_guard():
    with pytest.raises(pk.CtriError, match="SINGULAR"):
        pk.ctri_penta_factor_query(20, (0.0, 1.0, 1.0, 1.0, 0.0))  # mu_1 = d - l u / d = 0


def _run_block_pcr(alpha, gamma, fold, b, cyclic):
    P, q = b.shape[0], alpha.shape[0]
    b = b.copy()
    for k in range(q):
        s = 1 << k
        nb = b.copy()
        for i in range(P):
            im, ip = i - s, i + s
            if cyclic:
                im, ip = im % P, ip % P
            if im >= 0 and im < P:
                nb[i] -= alpha[k, i] @ b[im]
            if ip >= 0 and ip < P:
                nb[i] -= gamma[k, i] @ b[ip]
        b = nb
    return np.stack([fold[i] @ b[i] for i in range(P)])


@pytest.mark.parametrize("bands", PENTA_BANDS)
@pytest.mark.parametrize("P,cyclic", [(2, True), (4, True), (8, True), (16, True), (2, False), (3, False),
                                      (5, False), (8, False)])
def test_penta_block_pcr_vs_dense(bands, P, cyclic):
    """2x2-block PCR (+ fold) on the reduced system equals the dense solve of the Schur complement
    (the block matrix [L^, D^, U^] of the plan tables), for wide and narrow partitions."""
    for n in (8, 40):
        t = pk.ctri_penta_factor_query(n, bands)
        A = np.zeros((2 * P, 2 * P))
        for i in range(P):
            A[2 * i:2 * i + 2, 2 * i:2 * i + 2] += t["Dh"] if (cyclic or i > 0) else t["Dh_first"]
            if cyclic or i > 0:
                j = (i - 1) % P
                A[2 * i:2 * i + 2, 2 * j:2 * j + 2] += t["Lh"]
            if cyclic or i < P - 1:
                j = (i + 1) % P
                A[2 * i:2 * i + 2, 2 * j:2 * j + 2] += t["Uh"]
        a, g, f = pk.ctri_penta_block_pcr(P, n, bands, cyclic)
        assert a.shape[0] == math.ceil(math.log2(P))
        rng = np.random.default_rng(P + n)
        for _ in range(2):
            b = rng.uniform(-1, 1, (P, 2))
            x = _run_block_pcr(a, g, f, b, cyclic)
            assert np.max(np.abs(x.ravel() - np.linalg.solve(A, b.ravel()))) < 1e-13


def test_penta_block_pcr_rejects_cyclic_non_pow2():
    with pytest.raises(pk.CtriError, match="UNSUPPORTED"):
        pk.ctri_penta_block_pcr(3, 20, PENTA_BANDS[0], True)


@pytest.mark.parametrize("bands", PENTA_BANDS)
@pytest.mark.parametrize("P,cyclic", [(3, True), (5, True), (6, True), (7, True), (11, True), (2, True),
                                      (4, True), (8, True), (3, False), (6, False)])
def test_penta_reduced_schedule_vs_dense(bands, P, cyclic):
    """The block step schedule of the pentadiagonal reduced system -- block PCR, or for cyclic
    non-power-of-two P the paper's detach / PCR / fold / reattach with 2x2
    blocks -- equals the dense solve of the block matrix [L^, D^, U^]; its detach counts follow
    P:346 (P - 2^floor(log2 P) rows, popcount(P) - 1 stages)."""
    for n in (8, 40):
        t = pk.ctri_penta_factor_query(n, bands)
        A = np.zeros((2 * P, 2 * P))
        for i in range(P):
            A[2 * i:2 * i + 2, 2 * i:2 * i + 2] += t["Dh"] if (cyclic or i > 0) else t["Dh_first"]
            if cyclic or i > 0:
                j = (i - 1) % P
                A[2 * i:2 * i + 2, 2 * j:2 * j + 2] += t["Lh"]
            if cyclic or i < P - 1:
                j = (i + 1) % P
                A[2 * i:2 * i + 2, 2 * j:2 * j + 2] += t["Uh"]
        rng = np.random.default_rng(3 * P + n)
        for _ in range(2):
            b = rng.uniform(-1, 1, (P, 2))
            x, steps, ds, dr = pk.ctri_penta_reduced_schedule_apply(P, n, bands, b, cyclic)
            assert np.max(np.abs(x.ravel() - np.linalg.solve(A, b.ravel()))) < 1e-13
        if cyclic and P & (P - 1):
            q = int(math.floor(math.log2(P)))
            assert dr == P - 2 ** q and ds == bin(P).count("1") - 1
            assert steps == q + 1 + 2 * ds  # PCR stages, fold, detach and reattach levels
        else:
            assert ds == 0 and dr == 0 and steps == math.ceil(math.log2(P)) + 1


def test_scheme_coefficients_from_library():
    """ctri_scheme_coef (the binding only marshals): the collocated pair a = 14/9, b = 1/9 at
    alpha = 1/3 (R8) and the staggered schemes of P:202-206 (R18), against the oracle's
    independently written tables; unknown schemes and bad spacings are rejected."""
    import oracle
    from paper_2101_02286_b200 import CtriError, ctri
    h = 2 * math.pi / 64
    c, bd = ctri.ctri_scheme_coef(ctri.CTRI_SCHEME_COLLOCATED_D1, h)
    a, b = 14 / 9, 1 / 9
    assert np.allclose(c, (-b / (4 * h), -a / (2 * h), 0.0, a / (2 * h), b / (4 * h)), rtol=1e-15)
    assert bd == (1 / 3, 1.0, 1 / 3)
    c, bd = ctri.ctri_scheme_coef(ctri.CTRI_SCHEME_STAGGERED_D1, h)
    assert np.allclose(c, oracle.staggered_deriv_coef(h), rtol=1e-15) and bd == (9 / 62, 1.0, 9 / 62)
    c, bd = ctri.ctri_scheme_coef(ctri.CTRI_SCHEME_STAGGERED_I)
    assert np.allclose(c, oracle.staggered_interp_coef(), rtol=1e-15) and bd == (3 / 10, 1.0, 3 / 10)
    # Lele's sixth-order family at alpha = 1/3: a = (2/3)(alpha + 2), b = (1/3)(4 alpha - 1)
    c, _ = ctri.ctri_scheme_coef(ctri.CTRI_SCHEME_COLLOCATED_D1, 1.0)
    assert abs(2 * c[3] - (2 / 3) * (1 / 3 + 2)) < 1e-15 and abs(4 * c[4] - (4 / 3 - 1) / 3) < 1e-15
    for bad in ((7, 1.0), (ctri.CTRI_SCHEME_COLLOCATED_D1, 0.0), (ctri.CTRI_SCHEME_STAGGERED_D1, -1.0)):
        with pytest.raises(CtriError):
            ctri.ctri_scheme_coef(*bad)
