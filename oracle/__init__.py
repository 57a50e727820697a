"""CPU oracle for the batched cyclic tridiagonal solve (TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2101_02286_b200``) never imports it and shares no code,
tables or constants with it.

The arithmetic lives in ``ctri_oracle.c`` (plain C, fp64, OpenMP over batch
columns); this module only marshals numpy arrays into it.  See the C file's
header for the passages each function follows.  Every function here is
pinned by ``tests/test_oracle_pins.py`` against dense elimination and closed
forms (DESIGN.md section "Oracle and its pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ctri_oracle.c")
_LIB = os.path.join(_HERE, "libctri_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle shared library with gcc (-O3 as BASELINE.md section 3 specifies,
    OpenMP, no fast-math, no FMA contraction: the arithmetic is exactly the C source's)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-std=c11",
               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", _LIB, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64p = ctypes.POINTER(ctypes.c_int64)
        dp = ctypes.c_void_p
        lib.oracle_cyclic_solve.argtypes = [i64p, ctypes.c_int, dp, dp, dp]
        lib.oracle_acyclic_solve.argtypes = [i64p, ctypes.c_int, dp, dp, dp]
        lib.oracle_rhs_stencil.argtypes = [i64p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, dp, dp]
        lib.oracle_rhs_stencil5.argtypes = [i64p, ctypes.c_int, dp, dp, dp]
        lib.oracle_penta_solve.argtypes = [i64p, ctypes.c_int, dp, ctypes.c_int, dp, dp]
        lib.oracle_deriv.argtypes = [i64p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, dp, dp]
        for fn in (lib.oracle_cyclic_solve, lib.oracle_acyclic_solve, lib.oracle_rhs_stencil,
                   lib.oracle_rhs_stencil5, lib.oracle_penta_solve,
                   lib.oracle_deriv):
            fn.restype = ctypes.c_int
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _dims(shape):
    if len(shape) != 3:
        raise ValueError("oracle expects a 3D right-layout array")
    return (ctypes.c_int64 * 3)(*[int(s) for s in shape])


def _as3d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(a.shape[0], 1, 1)
    return a


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def cyclic_solve(b: np.ndarray, solve_dim: int = 0, bands=(1 / 3, 1.0, 1 / 3)) -> np.ndarray:
    """x = A^{-1} b along ``solve_dim`` of a 3D (or 1D) array; A cyclic, bands (l, d, u)."""
    shape = b.shape
    b3 = _as3d(b)
    sd = solve_dim if b.ndim == 3 else 0
    x = np.empty_like(b3)
    bnd = np.asarray(bands, dtype=np.float64)
    rc = _load().oracle_cyclic_solve(_dims(b3.shape), sd, bnd.ctypes.data, b3.ctypes.data,
                                     x.ctypes.data)
    if rc:
        raise ValueError("oracle_cyclic_solve: invalid argument")
    return x.reshape(shape)


def acyclic_solve(b: np.ndarray, solve_dim: int = 0, bands=(1 / 3, 1.0, 1 / 3)) -> np.ndarray:
    shape = b.shape
    b3 = _as3d(b)
    sd = solve_dim if b.ndim == 3 else 0
    x = np.empty_like(b3)
    bnd = np.asarray(bands, dtype=np.float64)
    rc = _load().oracle_acyclic_solve(_dims(b3.shape), sd, bnd.ctypes.data, b3.ctypes.data,
                                      x.ctypes.data)
    if rc:
        raise ValueError("oracle_acyclic_solve: invalid argument")
    return x.reshape(shape)


def rhs_stencil(f: np.ndarray, solve_dim: int, a: float, bc: float, h: float) -> np.ndarray:
    shape = f.shape
    f3 = _as3d(f)
    sd = solve_dim if f.ndim == 3 else 0
    out = np.empty_like(f3)
    rc = _load().oracle_rhs_stencil(_dims(f3.shape), sd, a, bc, h, f3.ctypes.data, out.ctypes.data)
    if rc:
        raise ValueError("oracle_rhs_stencil: invalid argument")
    return out.reshape(shape)


def penta_solve(b: np.ndarray, solve_dim: int = 0, bands=(0.05, 0.3, 1.0, 0.3, 0.05),
                cyclic: bool = True) -> np.ndarray:
    """x = A^{-1} b, A pentadiagonal with bands (e, l, d, u, f) = A[i, i-2..i+2] (r = 2)."""
    shape = b.shape
    b3 = _as3d(b)
    sd = solve_dim if b.ndim == 3 else 0
    x = np.empty_like(b3)
    bnd = np.ascontiguousarray(bands, dtype=np.float64)
    if bnd.shape != (5,):
        raise ValueError("bands must be (e, l, d, u, f)")
    rc = _load().oracle_penta_solve(_dims(b3.shape), sd, bnd.ctypes.data, int(bool(cyclic)),
                                    b3.ctypes.data, x.ctypes.data)
    if rc:
        raise ValueError("oracle_penta_solve: invalid argument")
    return x.reshape(shape)


def rhs_stencil5(f: np.ndarray, solve_dim: int, coef) -> np.ndarray:
    """b_j = sum_{k=-2..2} coef[k+2] f_{(j+k) mod N} along solve_dim (P:202-206 schemes)."""
    shape = f.shape
    f3 = _as3d(f)
    sd = solve_dim if f.ndim == 3 else 0
    c = np.ascontiguousarray(coef, dtype=np.float64)
    if c.shape != (5,):
        raise ValueError("coef must hold 5 values (offsets -2..2)")
    out = np.empty_like(f3)
    rc = _load().oracle_rhs_stencil5(_dims(f3.shape), sd, c.ctypes.data, f3.ctypes.data,
                                     out.ctypes.data)
    if rc:
        raise ValueError("oracle_rhs_stencil5: invalid argument")
    return out.reshape(shape)


def compact_apply(f: np.ndarray, solve_dim: int, coef, bands) -> np.ndarray:
    """A compact scheme: the five-point RHS, then x = A^{-1} rhs with cyclic `bands`."""
    return cyclic_solve(rhs_stencil5(f, solve_dim, coef), solve_dim, bands)


# The staggered sixth-order schemes of PAPER.md P:202-206, with half-node values
# g_i = f_{i+1/2} stored at index i (so f_{i-1/2} = g_{i-1}, f_{i+3/2} = g_{i+1}, ...).
#   9/62 f'_{i-1} + f'_i + 9/62 f'_{i+1} = 63/62 (f_{i+1/2}-f_{i-1/2})/D + 17/62 (f_{i+3/2}-f_{i-3/2})/(3D)
#   3/10 fI_{i-1} + fI_i + 3/10 fI_{i+1} = 3/2 (f_{i+1/2}+f_{i-1/2})/2 + 1/10 (f_{i+3/2}+f_{i-3/2})/2
STAGGERED_DERIV_ALPHA = 9.0 / 62.0
STAGGERED_INTERP_ALPHA = 3.0 / 10.0


def staggered_deriv_coef(delta: float):
    """Offsets -2..2 of the staggered-derivative RHS in the g-indexing."""
    a, b = 63.0 / 62.0, 17.0 / 62.0
    return [-b / (3 * delta), -a / delta, a / delta, b / (3 * delta), 0.0]


def staggered_interp_coef():
    """Offsets -2..2 of the staggered-interpolation RHS in the g-indexing."""
    a, b = 3.0 / 2.0, 1.0 / 10.0
    return [b / 2, a / 2, a / 2, b / 2, 0.0]


def deriv(f: np.ndarray, solve_dim: int = 0, alpha: float = 1 / 3, a: float = 14 / 9,
          bc: float = 1 / 9, h: float | None = None) -> np.ndarray:
    """Compact first derivative (stencil + cyclic solve); h defaults to 2*pi/N."""
    shape = f.shape
    f3 = _as3d(f)
    sd = solve_dim if f.ndim == 3 else 0
    if h is None:
        h = 2.0 * np.pi / f3.shape[sd]
    out = np.empty_like(f3)
    rc = _load().oracle_deriv(_dims(f3.shape), sd, alpha, a, bc, h, f3.ctypes.data,
                              out.ctypes.data)
    if rc:
        raise ValueError("oracle_deriv: invalid argument")
    return out.reshape(shape)
