"""Pins for the CPU oracle (oracle/ctri_oracle.c) against things other than itself.

Each test checks the oracle against what the paper and the mathematics fix:
dense Gaussian elimination (LAPACK dgesv via numpy) on the assembled matrix,
Cramer's rule on 3x3, the Fourier eigenvalues of the circulant A, the periodic
Green's function, the constant RHS, and the modified wavenumber of the compact
scheme (tests/golden/modified_wavenumber.txt).  Non-symmetric bands (l != u)
are used wherever the closed form allows, so a transposed band, a dropped
corner or a wrong sign fails.
"""
import math
import os

import numpy as np
import pytest

import oracle
import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
BANDS = [(0.2, 1.1, 0.4), (-0.3, 1.0, 0.25), (1 / 3, 1.0, 1 / 3), (0.45, 1.0, 0.45),
         (0.1, -0.9, 0.35)]


def dense_cyclic(N, bands):
    l, d, u = bands
    A = np.zeros((N, N))
    for i in range(N):
        A[i, i] += d
        A[i, (i - 1) % N] += l
        A[i, (i + 1) % N] += u
    return A


def dense_acyclic(N, bands):
    l, d, u = bands
    A = np.diag(np.full(N, d))
    A += np.diag(np.full(N - 1, l), -1) + np.diag(np.full(N - 1, u), 1)
    return A


def columns(arr, sd):
    """(N, ncols) view of a 3D array with the solve dim first."""
    return np.moveaxis(arr, sd, 0).reshape(arr.shape[sd], -1)


@pytest.mark.parametrize("N", [3, 4, 5, 8, 13, 64])
@pytest.mark.parametrize("bands", BANDS)
@pytest.mark.parametrize("sd", [0, 1, 2])
def test_oracle_vs_dense_ge(N, bands, sd):
    shape = [3, 5, 2]
    shape[sd] = N
    b = workloads.uniform(shape, 6)
    x = oracle.cyclic_solve(b, sd, bands)
    A = dense_cyclic(N, bands)
    xd = np.linalg.solve(A, columns(b, sd))
    xo = columns(x, sd)
    err = np.max(np.abs(xo - xd)) / np.max(np.abs(xd))
    assert err < 1e-13, err


@pytest.mark.parametrize("N", [1, 2, 3, 7, 64])
@pytest.mark.parametrize("bands", BANDS[:3])
def test_oracle_acyclic_vs_dense(N, bands):
    b = workloads.uniform((N, 4, 3), 7)
    x = oracle.acyclic_solve(b, 0, bands)
    xd = np.linalg.solve(dense_acyclic(N, bands), b.reshape(N, -1))
    assert np.max(np.abs(x.reshape(N, -1) - xd)) < 1e-13 * max(1.0, np.max(np.abs(xd)))


def test_oracle_cramer_3x3():
    """Brute force: Cramer's rule in pure Python on the 3x3 cyclic system."""
    l, d, u = 0.2, 1.1, 0.4
    A = [[d, u, l], [l, d, u], [u, l, d]]  # row 0: d x0 + u x1 + l x2 (corner A[0,2] = l)

    def det3(M):
        return (M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1])
                - M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0])
                + M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]))

    rhs = [0.7, -0.2, 0.5]
    D = det3(A)
    xs = []
    for c in range(3):
        M = [row[:] for row in A]
        for r in range(3):
            M[r][c] = rhs[r]
        xs.append(det3(M) / D)
    x = oracle.cyclic_solve(np.array(rhs), 0, (l, d, u))
    assert np.allclose(x, xs, rtol=0, atol=1e-15)


@pytest.mark.parametrize("N", [64, 8192])
def test_oracle_fourier_eigenvectors(N):
    """b_j = cos(2 pi k j / N) => x_j = b_j / (1 + 2 alpha cos(2 pi k / N)) (circulant A)."""
    alpha = 1 / 3
    ks = range(N) if N <= 64 else [0, 1, 2, 3, 1000, 4095, 4096, 4097, 8191]
    for k in ks:
        b = workloads.fourier_mode((N, 1, 1), 0, k)
        x = oracle.cyclic_solve(b, 0, (alpha, 1.0, alpha))
        expect = b / (1.0 + 2.0 * alpha * math.cos(2.0 * math.pi * k / N))
        assert np.max(np.abs(x - expect)) < 4e-15, (k, np.max(np.abs(x - expect)))
    # k = 0 -> 3/5 b ; Nyquist k = N/2 -> 3 b
    b = workloads.fourier_mode((N, 1, 1), 0, N // 2)
    assert np.max(np.abs(oracle.cyclic_solve(b, 0) - 3.0 * b)) < 4e-15


@pytest.mark.parametrize("alpha", [1 / 3, 0.45])
@pytest.mark.parametrize("N", [16, 64, 8192])
def test_oracle_green_function(alpha, N):
    """b = e_r => x_j = (lam^dlt + lam^(N-dlt)) / (sqrt(1-4a^2)(1-lam^N)), dlt = (j-r) mod N."""
    lam = (-1.0 + math.sqrt(1.0 - 4.0 * alpha * alpha)) / (2.0 * alpha)
    for r in sorted({0, 1, N // 2 - 1, N // 2, N - 1}):
        b = workloads.delta((N, 1, 1), 0, r)
        x = oracle.cyclic_solve(b, 0, (alpha, 1.0, alpha)).ravel()
        dl = (np.arange(N) - r) % N
        expect = (lam ** dl + lam ** (N - dl)) / (math.sqrt(1 - 4 * alpha ** 2) * (1 - lam ** N))
        assert np.max(np.abs(x - expect)) < 2e-15, (r, np.max(np.abs(x - expect)))


def test_oracle_constant_rhs():
    """b = 1 => x = 1/(1 + 2 alpha) = 3/5 ; and A 1 = 5/3 (row sums)."""
    b = np.ones((64, 4, 4))
    for sd in range(3):
        x = oracle.cyclic_solve(b, sd)
        assert np.max(np.abs(x - 0.6)) < 1e-15
    A = dense_cyclic(64, (1 / 3, 1, 1 / 3))
    assert np.allclose(A @ np.ones(64), 5 / 3, rtol=0, atol=1e-15)


def test_oracle_residual_large():
    """Residual ||Ax-b||_inf/||b||_inf at N = 8192 (band matvec, no dense matrix)."""
    b = workloads.uniform((8192, 3, 2), 2)
    x = oracle.cyclic_solve(b, 0)
    a = 1 / 3
    r = a * np.roll(x, 1, axis=0) + x + a * np.roll(x, -1, axis=0) - b
    assert np.max(np.abs(r)) / np.max(np.abs(b)) < 1e-15


def _golden_wavenumbers():
    rows = []
    with open(os.path.join(GOLDEN, "modified_wavenumber.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            N, k, kp = line.split()
            rows.append((int(N), int(k), float(kp)))
    return rows


def test_closed_form_wavenumber_matches_golden():
    """The closed form used below reproduces the tabulated values (guards the test itself)."""
    for N, k, kp in _golden_wavenumbers():
        h = 2 * math.pi / N
        val = (14 / 9 * math.sin(k * h) + (1 / 9) / 2 * math.sin(2 * k * h)) / (1 + 2 / 3 * math.cos(k * h)) / h
        assert abs(val - kp) < 1e-11


@pytest.mark.parametrize("sd", [0, 2])
def test_oracle_deriv_modified_wavenumber(sd):
    """O-DERIV on sin(kappa x) returns exactly k'(kappa) cos(kappa x) (golden table)."""
    for N, k, kp in _golden_wavenumbers():
        shape = [2, 3, 2]
        shape[sd] = N
        j = np.arange(N, dtype=np.int64)
        xs = 2 * math.pi * ((k * j) % N) / N
        sh = [1, 1, 1]
        sh[sd] = N
        f = np.broadcast_to(np.sin(xs).reshape(sh), shape).copy()
        df = oracle.deriv(f, sd)
        expect = kp * np.cos(xs).reshape(sh)
        assert np.max(np.abs(df - expect)) < 1e-12 * max(1.0, kp), (N, k)


def test_oracle_stencil_trig_identity():
    """Stencil on sin(kx): (a sin(kh)/h + b sin(2kh)/(2h)) cos(kx) exactly; constant -> 0."""
    N, k = 128, 9
    h = 2 * math.pi / N
    x = 2 * math.pi * np.arange(N) / N
    f = np.sin(k * x).reshape(N, 1, 1)
    r = oracle.rhs_stencil(f, 0, 14 / 9, 1 / 9, h).ravel()
    expect = (14 / 9 * math.sin(k * h) / h + (1 / 9) * math.sin(2 * k * h) / (2 * h)) * np.cos(k * x)
    assert np.max(np.abs(r - expect)) < 1e-12
    assert np.max(np.abs(oracle.rhs_stencil(np.full((N, 2, 2), 3.7), 0, 14 / 9, 1 / 9, h))) == 0.0


def test_oracle_deriv_order_and_conservation():
    """Sixth-order convergence for sin(x) and zero periodic sum."""
    errs = []
    for N in (16, 32, 64):
        x = 2 * math.pi * np.arange(N) / N
        f = np.sin(x).reshape(N, 1, 1)
        df = oracle.deriv(f, 0).ravel()
        errs.append(np.max(np.abs(df - np.cos(x))))
        assert abs(df.sum()) < 1e-12
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(5.5 <= o <= 6.5 for o in orders), orders


def test_oracle_layout_permutation():
    """Solving along dim 1 / 2 of a permuted array equals the dim-0 result permuted."""
    b0 = workloads.uniform((32, 6, 4), 2)
    x0 = oracle.cyclic_solve(b0, 0)
    b1 = np.ascontiguousarray(np.transpose(b0, (1, 0, 2)))
    x1 = oracle.cyclic_solve(b1, 1)
    b2 = np.ascontiguousarray(np.transpose(b0, (1, 2, 0)))
    x2 = oracle.cyclic_solve(b2, 2)
    assert np.array_equal(np.transpose(x1, (1, 0, 2)), x0)
    assert np.max(np.abs(np.transpose(x2, (2, 0, 1)) - x0)) < 1e-15


def test_oracle_rejects_bad_args():
    with pytest.raises(ValueError):
        oracle.cyclic_solve(np.ones((2, 3, 3)), 0)


# ---- staggered sixth-order schemes ----
def _half_node_mode(N, k, fn):
    """fn(kappa x_{i+1/2}) with x = 2 pi (i + 1/2)/N, the argument reduced in integers."""
    i = np.arange(N, dtype=np.int64)
    return fn(math.pi * ((k * (2 * i + 1)) % (2 * N)) / N)


def _node_mode(N, k, fn):
    i = np.arange(N, dtype=np.int64)
    return fn(2 * math.pi * ((k * i) % N) / N)


def test_stencil5_matches_dense_circulant():
    """rhs_stencil5 equals the dense circulant product C f with C[j, j+k mod N] = c_k (N = 7)."""
    N = 7
    coef = [0.3, -1.7, 0.25, 2.1, -0.6]
    C = np.zeros((N, N))
    for j in range(N):
        for k in range(-2, 3):
            C[j, (j + k) % N] += coef[k + 2]
    f = workloads.uniform((N, 3, 2), 11)
    got = oracle.rhs_stencil5(f, 0, coef)
    expect = np.einsum("jk,kab->jab", C, f)
    assert np.max(np.abs(got - expect)) < 1e-15
    got2 = oracle.rhs_stencil5(np.ascontiguousarray(np.transpose(f, (1, 2, 0))), 2, coef)
    assert np.max(np.abs(np.transpose(got2, (2, 0, 1)) - expect)) < 1e-15


def test_stencil5_reduces_to_collocated():
    """The collocated derivative stencil is the 5-point stencil (-b/4h, -a/2h, 0, a/2h, b/4h)."""
    N = 32
    h = 2 * math.pi / N
    f = workloads.uniform((N, 4, 3), 12)
    a, b = 14 / 9, 1 / 9
    got = oracle.rhs_stencil5(f, 0, [-b / (4 * h), -a / (2 * h), 0.0, a / (2 * h), b / (4 * h)])
    assert np.max(np.abs(got - oracle.rhs_stencil(f, 0, a, b, h))) < 1e-13


@pytest.mark.parametrize("N,k", [(64, 1), (64, 5), (64, 17), (64, 31), (128, 40), (30, 7)])
def test_staggered_deriv_modified_wavenumber(N, k):
    """Fourier analysis of P:203-204 with g_i = sin(k x_{i+1/2}):
    f'_i = k'(k) cos(k x_i),  k' h = [2a sin(kh/2) + (2b/3) sin(3kh/2)] / (1 + 2 alpha cos kh)."""
    h = 2 * math.pi / N
    g = _half_node_mode(N, k, np.sin).reshape(N, 1, 1)
    df = oracle.compact_apply(g, 0, oracle.staggered_deriv_coef(h),
                              (oracle.STAGGERED_DERIV_ALPHA, 1.0, oracle.STAGGERED_DERIV_ALPHA))
    kp = (2 * 63 / 62 * math.sin(k * h / 2) + 2 * 17 / 62 / 3 * math.sin(3 * k * h / 2)) / (
        1 + 2 * 9 / 62 * math.cos(k * h)) / h
    assert np.max(np.abs(df.ravel() - kp * _node_mode(N, k, np.cos))) < 1e-13 * max(1.0, kp)


@pytest.mark.parametrize("N,k", [(64, 0), (64, 3), (64, 20), (64, 32), (30, 11)])
def test_staggered_interp_transfer_function(N, k):
    """Fourier analysis of P:205-206 with g_i = cos(k x_{i+1/2}):
    fI_i = T(k) cos(k x_i),  T = [a cos(kh/2) + b cos(3kh/2)] / (1 + 2 alpha cos kh)."""
    h = 2 * math.pi / N
    g = _half_node_mode(N, k, np.cos).reshape(N, 1, 1)
    fi = oracle.compact_apply(g, 0, oracle.staggered_interp_coef(),
                              (oracle.STAGGERED_INTERP_ALPHA, 1.0, oracle.STAGGERED_INTERP_ALPHA))
    T = (1.5 * math.cos(k * h / 2) + 0.1 * math.cos(3 * k * h / 2)) / (1 + 0.6 * math.cos(k * h))
    assert np.max(np.abs(fi.ravel() - T * _node_mode(N, k, np.cos))) < 1e-14
    if k == N // 2:  # Nyquist: cos(k x_{i+1/2}) = 0 exactly, the interpolant is 0
        assert abs(T) < 1e-15


@pytest.mark.parametrize("which", ["deriv", "interp"])
def test_staggered_sixth_order(which):
    """Both staggered schemes converge at sixth order on exp(sin x) (P:201 'sixth order')."""
    errs = []
    for N in (16, 32, 64):
        h = 2 * math.pi / N
        xh = h * (np.arange(N) + 0.5)
        xn = h * np.arange(N)
        g = np.exp(np.sin(xh)).reshape(N, 1, 1)
        if which == "deriv":
            out = oracle.compact_apply(g, 0, oracle.staggered_deriv_coef(h),
                                       (9 / 62, 1.0, 9 / 62)).ravel()
            exact = np.cos(xn) * np.exp(np.sin(xn))
        else:
            out = oracle.compact_apply(g, 0, oracle.staggered_interp_coef(),
                                       (3 / 10, 1.0, 3 / 10)).ravel()
            exact = np.exp(np.sin(xn))
        errs.append(np.max(np.abs(out - exact)))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(5.5 <= o <= 7.0 for o in orders), (which, orders, errs)


# ---- pentadiagonal (r = 2) oracle: PAPER.md P:212 (w = 5), SURVEY 8(f) N3 ----
PENTA_BANDS = [(0.05, 0.3, 1.0, 0.3, 0.05),          # symmetric, diagonally dominant
               (-0.07, 0.21, 1.3, -0.33, 0.11),      # non-symmetric
               (1 / 20, 1 / 2, 1.0, 1 / 2, 1 / 20)]  # Lele's tenth-order LHS (beta, alpha)


def _dense_penta(N, bands, cyclic):
    e, l, d, u, f = bands
    A = np.zeros((N, N))
    for i in range(N):
        for off, v in ((-2, e), (-1, l), (0, d), (1, u), (2, f)):
            j = i + off
            if 0 <= j < N:
                A[i, j] += v
            elif cyclic:
                A[i, j % N] += v
    return A


@pytest.mark.parametrize("bands", PENTA_BANDS)
@pytest.mark.parametrize("cyclic", [True, False])
@pytest.mark.parametrize("N", [5, 6, 7, 8, 11, 32, 64])
def test_penta_oracle_vs_dense(bands, cyclic, N):
    """Dense LAPACK solve of the explicitly assembled (cyclic) pentadiagonal matrix."""
    b = workloads.uniform((N, 3, 2), 50 + N)
    x = oracle.penta_solve(b, 0, bands, cyclic)
    A = _dense_penta(N, bands, cyclic)
    expect = np.einsum("ij,jab->iab", np.linalg.inv(A), b)
    assert np.max(np.abs(x - expect)) < 1e-14 * max(1.0, np.max(np.abs(expect)))


@pytest.mark.parametrize("bands", PENTA_BANDS)
@pytest.mark.parametrize("N,k", [(64, 0), (64, 5), (64, 32), (1024, 77), (1000, 333)])
def test_penta_oracle_fourier_eigenvector(bands, N, k):
    """b_j = cos(theta j) => x_j = Re(e^{i theta j} / lambda(theta)),
    lambda = d + l e^{-i theta} + u e^{i theta} + e e^{-2 i theta} + f e^{2 i theta}."""
    e, l, d, u, f = bands
    th = 2 * math.pi * k / N
    lam = d + l * np.exp(-1j * th) + u * np.exp(1j * th) + e * np.exp(-2j * th) + f * np.exp(2j * th)
    j = np.arange(N, dtype=np.int64)
    ph = 2 * math.pi * ((k * j) % N) / N
    b = np.cos(ph).reshape(N, 1, 1)
    x = oracle.penta_solve(np.broadcast_to(b, (N, 2, 3)).copy(), 0, bands, True)
    expect = np.real(np.exp(1j * ph) / lam).reshape(N, 1, 1)
    assert np.max(np.abs(x - expect)) < 1e-14


def test_penta_oracle_reduces_to_tridiagonal():
    """e = f = 0: the pentadiagonal oracle equals the (pinned) tridiagonal one, both layouts."""
    b = workloads.uniform((40, 5, 6), 61)
    for sd in (0, 1, 2):
        for cyc in (True, False):
            x5 = oracle.penta_solve(b, sd, (0.0, 0.2, 1.1, 0.4, 0.0), cyc)
            x3 = (oracle.cyclic_solve if cyc else oracle.acyclic_solve)(b, sd, (0.2, 1.1, 0.4))
            assert np.max(np.abs(x5 - x3)) < 1e-15


def test_penta_oracle_layout_permutation():
    b0 = workloads.uniform((48, 6, 4), 62)
    x0 = oracle.penta_solve(b0, 0, PENTA_BANDS[1], True)
    x2 = oracle.penta_solve(np.ascontiguousarray(np.transpose(b0, (1, 2, 0))), 2, PENTA_BANDS[1], True)
    assert np.max(np.abs(np.transpose(x2, (2, 0, 1)) - x0)) < 1e-15
