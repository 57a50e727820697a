"""Thin ctypes binding of ``include/ctri.h`` (argument marshalling only).

Every step of the solve runs inside ``libctri.so`` (sm_100a kernels + NCCL).
This module converts torch tensors / numpy arrays to pointers, checks status
codes and raises :class:`CtriError`.  There is no CPU fallback: if the
extension is missing the import fails loudly.

Function names mirror the C ABI (``ctri_plan_create``, ``ctri_solve`` ...);
:class:`Plan` and :class:`LoopbackGroup` are small conveniences over them.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libctri.so")

CTRI_FLAG_FULL_BACKSUB = 1 << 0
CTRI_FLAG_GENERIC_LOCAL = 1 << 1
CTRI_FLAG_TIMING = 1 << 2
CTRI_FLAG_DERIV = 1 << 3
CTRI_FLAG_NCCL_ROUNDS = 1 << 4
CTRI_FLAG_ALLGATHER = 1 << 5
CTRI_FLAG_FUSED_REDUCED = 1 << 6
CTRI_MAX_STAGES = 16
ABI_VERSION = 6

STATUS = {0: "CTRI_OK", 1: "CTRI_ERR_INVALID_ARG", 2: "CTRI_ERR_UNSUPPORTED", 3: "CTRI_ERR_SINGULAR",
          4: "CTRI_ERR_PARTITION_TOO_SMALL", 5: "CTRI_ERR_CUDA", 6: "CTRI_ERR_NCCL",
          7: "CTRI_ERR_OOM"}

# Every symbol include/ctri.h declares (checked by tests/test_abi.py).
ABI_SYMBOLS = ("ctri_status_string", "ctri_last_error", "ctri_abi_version", "ctri_get_unique_id",
               "ctri_plan_create", "ctri_plan_create_loopback", "ctri_solve", "ctri_solve_loopback",
               "ctri_solve_host", "ctri_deriv", "ctri_deriv_loopback", "ctri_get_stats",
               "ctri_plan_destroy", "ctri_factor_query", "ctri_pcr_coefficients",
               "ctri_reduced_schedule", "ctri_compact_apply", "ctri_compact_apply_loopback",
               "ctri_reduced_inverse", "ctri_plan_create_penta", "ctri_plan_create_penta_loopback",
               "ctri_penta_factor_query", "ctri_penta_block_pcr", "ctri_scheme_coef",
               "ctri_penta_reduced_schedule_apply")


class CtriError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        self.name = STATUS.get(status, f"status {status}")
        super().__init__(f"{where}: {self.name}: {detail}")


class ctri_stats(ctypes.Structure):
    _fields_ = [("global_dims", ctypes.c_int64 * 3),
                ("solve_dim", ctypes.c_int32), ("nparts", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("cyclic", ctypes.c_int32),
                ("n_local", ctypes.c_int64), ("m_batch", ctypes.c_int64),
                ("local_kernel", ctypes.c_int32), ("rows_per_thread", ctypes.c_int32),
                ("cluster_size", ctypes.c_int32), ("tile_columns", ctypes.c_int32),
                ("chunk_heads", ctypes.c_int32), ("window_rows", ctypes.c_int32),
                ("pcr_stages", ctypes.c_int32), ("comm_rounds", ctypes.c_int32),
                ("sends_per_solve", ctypes.c_int32),
                ("bytes_sent_per_solve", ctypes.c_int64),
                ("launches_per_solve", ctypes.c_int32),
                ("solves", ctypes.c_uint64),
                ("t_total_us", ctypes.c_float), ("t_local_us", ctypes.c_float),
                ("t_yexchange_us", ctypes.c_float), ("t_bhat_us", ctypes.c_float),
                ("t_stage_us", ctypes.c_float * CTRI_MAX_STAGES),
                ("t_xexchange_us", ctypes.c_float), ("t_backsub_us", ctypes.c_float),
                ("tile_variant", ctypes.c_int32), ("tile_stages", ctypes.c_int32),
                ("reduced_path", ctypes.c_int32), ("device_error", ctypes.c_int32),
                ("vparts", ctypes.c_int32), ("grid_ctas", ctypes.c_int32),
                ("detach_stages", ctypes.c_int32), ("detached_rows", ctypes.c_int32),
                ("band_halfwidth", ctypes.c_int32),
                ("t_reduced_kernel_us", ctypes.c_float), ("t_window_us", ctypes.c_float),
                ("t_p2p_y_us", ctypes.c_float), ("t_p2p_step_us", ctypes.c_float * CTRI_MAX_STAGES),
                ("t_p2p_x_us", ctypes.c_float), ("p2p_steps", ctypes.c_int32),
                ("p2p_epoch", ctypes.c_uint32), ("reduced_rows", ctypes.c_int32),
                ("vchain", ctypes.c_int32), ("halo_epoch", ctypes.c_uint32)]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            if hasattr(v, "__len__"):
                v = list(v)
            d[name] = v
        d["t_stage_us"] = d["t_stage_us"][: max(0, self.pcr_stages)]
        d["t_p2p_step_us"] = d["t_p2p_step_us"][: max(0, self.p2p_steps)]
        return d


_lib = None


def load(build_if_missing: bool = False):
    """Load libctri.so (raises if it is missing; optionally builds it first)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if build_if_missing:
            from . import build as _b
            _b.build()
        else:
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2101_02286_b200.build`")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i64p = ctypes.POINTER(ctypes.c_int64)
    dp = ctypes.POINTER(ctypes.c_double)
    st = ctypes.c_int
    sig = {
        "ctri_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "ctri_last_error": (ctypes.c_char_p, []),
        "ctri_abi_version": (ctypes.c_int, []),
        "ctri_get_unique_id": (st, [P]),
        "ctri_plan_create": (st, [ctypes.POINTER(P), i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  dp, ctypes.c_int, P, ctypes.c_uint32, P]),
        "ctri_plan_create_loopback": (st, [ctypes.POINTER(P), ctypes.c_int, i64p, ctypes.c_int, dp,
                                           ctypes.c_int, ctypes.c_uint32, P]),
        "ctri_solve": (st, [P, P, P, P]),
        "ctri_solve_loopback": (st, [ctypes.POINTER(P), ctypes.c_int, ctypes.POINTER(P),
                                     ctypes.POINTER(P), P]),
        "ctri_solve_host": (st, [P, P, P, P]),
        "ctri_deriv": (st, [P, P, P, ctypes.c_double, ctypes.c_double, ctypes.c_double, P]),
        "ctri_deriv_loopback": (st, [ctypes.POINTER(P), ctypes.c_int, ctypes.POINTER(P),
                                     ctypes.POINTER(P), ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, P]),
        "ctri_compact_apply": (st, [P, dp, P, P, P]),
        "ctri_scheme_coef": (st, [ctypes.c_int, ctypes.c_double, dp, dp]),
        "ctri_reduced_inverse": (st, [ctypes.c_int, ctypes.c_int, dp, dp, dp, dp]),
        "ctri_plan_create_penta": (st, [ctypes.POINTER(P), i64p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        dp, ctypes.c_int, P, ctypes.c_uint32, P]),
        "ctri_plan_create_penta_loopback": (st, [ctypes.POINTER(P), ctypes.c_int, i64p, ctypes.c_int, dp,
                                                 ctypes.c_int, ctypes.c_uint32, P]),
        "ctri_penta_factor_query": (st, [ctypes.c_int64, dp, dp, dp, ctypes.POINTER(ctypes.c_int)]),
        "ctri_penta_block_pcr": (st, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, dp, ctypes.c_int, dp, dp, dp,
                                      ctypes.POINTER(ctypes.c_int)]),
        "ctri_penta_reduced_schedule_apply": (st, [ctypes.c_int, ctypes.c_int, ctypes.c_int64, dp, dp, dp,
                                                   ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                                   ctypes.POINTER(ctypes.c_int)]),
        "ctri_compact_apply_loopback": (st, [ctypes.POINTER(P), ctypes.c_int, dp, ctypes.POINTER(P),
                                             ctypes.POINTER(P), P]),
        "ctri_get_stats": (st, [P, ctypes.POINTER(ctri_stats)]),
        "ctri_plan_destroy": (st, [P]),
        "ctri_factor_query": (st, [ctypes.c_int64, dp, dp, dp, dp, ctypes.POINTER(ctypes.c_int)]),
        "ctri_pcr_coefficients": (st, [ctypes.c_int, ctypes.c_int, dp, dp, dp, dp, dp, dp,
                                       ctypes.POINTER(ctypes.c_int)]),
        "ctri_reduced_schedule": (st, [ctypes.c_int, ctypes.c_int, dp, dp, dp, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), dp,
                                       ctypes.POINTER(ctypes.c_int), dp,
                                       ctypes.POINTER(ctypes.c_int)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ctri_abi_version() != ABI_VERSION:
        raise ImportError("libctri.so ABI version mismatch; rebuild")
    _lib = lib
    return lib


def _check(status: int, where: str):
    if status != 0:
        detail = load().ctri_last_error().decode(errors="replace")
        raise CtriError(status, where, detail)


def _ptr(t) -> int:
    """Device/host address of a torch tensor, numpy array or int."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"] or t.dtype != np.float64:
            raise ValueError("numpy buffers must be C-contiguous float64")
        return t.ctypes.data
    # torch tensor
    if not t.is_contiguous() or str(t.dtype) != "torch.float64":
        raise ValueError("tensors must be contiguous float64")
    return t.data_ptr()


def _dev(t, numel: int, what: str):
    """Plan / LoopbackGroup wrappers: a CUDA float64 tensor holding exactly the local slab."""
    if isinstance(t, int):
        return t
    if isinstance(t, np.ndarray) or not getattr(t, "is_cuda", False):
        raise ValueError(f"{what}: expected a CUDA tensor (device memory), got {type(t).__name__}"
                         f"{'' if isinstance(t, np.ndarray) else ' on ' + str(getattr(t, 'device', '?'))}")
    if t.numel() != numel:
        raise ValueError(f"{what}: {t.numel()} elements, the plan's local slab has {numel}")
    return t


def _host(t, numel: int, what: str):
    if isinstance(t, int):
        return t
    if getattr(t, "is_cuda", False):
        raise ValueError(f"{what}: expected host memory")
    n = t.size if isinstance(t, np.ndarray) else t.numel()
    if n != numel:
        raise ValueError(f"{what}: {n} elements, the plan's local slab has {numel}")
    return t


def _stream_ptr(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dbl3(v):
    return (ctypes.c_double * 3)(*[float(x) for x in v])


# ---------------------------------------------------------------- raw ABI (same names)
def ctri_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().ctri_get_unique_id(buf), "ctri_get_unique_id")
    return buf.raw


def ctri_plan_create(global_dims, solve_dim, nparts=1, rank=0, bands=(1 / 3, 1.0, 1 / 3), cyclic=True,
                     unique_id: bytes | None = None, flags: int = 0, stream=None) -> int:
    h = ctypes.c_void_p()
    dims = (ctypes.c_int64 * 3)(*[int(d) for d in global_dims])
    uid = ctypes.create_string_buffer(unique_id, 128) if unique_id is not None else None
    _check(load().ctri_plan_create(ctypes.byref(h), dims, int(solve_dim), int(nparts), int(rank),
                                   _dbl3(bands), int(bool(cyclic)), uid, int(flags),
                                   _stream_ptr(stream)), "ctri_plan_create")
    return h.value


def ctri_plan_create_loopback(global_dims, solve_dim, nparts, bands=(1 / 3, 1.0, 1 / 3), cyclic=True,
                              flags: int = 0, stream=None) -> list[int]:
    hs = (ctypes.c_void_p * nparts)()
    dims = (ctypes.c_int64 * 3)(*[int(d) for d in global_dims])
    _check(load().ctri_plan_create_loopback(hs, int(nparts), dims, int(solve_dim), _dbl3(bands),
                                            int(bool(cyclic)), int(flags), _stream_ptr(stream)),
           "ctri_plan_create_loopback")
    return [hs[i] for i in range(nparts)]


def _dbl5(v):
    if len(v) != 5:
        raise ValueError("pentadiagonal bands must be (e, l, d, u, f)")
    return (ctypes.c_double * 5)(*[float(x) for x in v])


def ctri_plan_create_penta(global_dims, solve_dim, nparts=1, rank=0, bands=(0.05, 0.3, 1.0, 0.3, 0.05),
                           cyclic=True, unique_id: bytes | None = None, flags: int = 0, stream=None) -> int:
    h = ctypes.c_void_p()
    dims = (ctypes.c_int64 * 3)(*[int(d) for d in global_dims])
    uid = ctypes.create_string_buffer(unique_id, 128) if unique_id is not None else None
    _check(load().ctri_plan_create_penta(ctypes.byref(h), dims, int(solve_dim), int(nparts), int(rank),
                                         _dbl5(bands), int(bool(cyclic)), uid, int(flags),
                                         _stream_ptr(stream)), "ctri_plan_create_penta")
    return h.value


def ctri_plan_create_penta_loopback(global_dims, solve_dim, nparts, bands=(0.05, 0.3, 1.0, 0.3, 0.05),
                                    cyclic=True, flags: int = 0, stream=None) -> list[int]:
    hs = (ctypes.c_void_p * nparts)()
    dims = (ctypes.c_int64 * 3)(*[int(d) for d in global_dims])
    _check(load().ctri_plan_create_penta_loopback(hs, int(nparts), dims, int(solve_dim), _dbl5(bands),
                                                  int(bool(cyclic)), int(flags), _stream_ptr(stream)),
           "ctri_plan_create_penta_loopback")
    return [hs[i] for i in range(nparts)]


def ctri_penta_factor_query(n: int, bands):
    """Host-only: S0, S1, R0, R1 (n-2 each), the 2x2 blocks L^, D^, U^, D^(first) and the window."""
    N = n - 2
    SR = np.zeros(4 * max(1, N))
    hat = np.zeros(16)
    w = ctypes.c_int()
    dp = ctypes.POINTER(ctypes.c_double)
    _check(load().ctri_penta_factor_query(int(n), _dbl5(bands), SR.ctypes.data_as(dp),
                                          hat.ctypes.data_as(dp), ctypes.byref(w)),
           "ctri_penta_factor_query")
    S = SR[:2 * N].reshape(2, N).T.copy()
    R = SR[2 * N:].reshape(2, N).T.copy()
    blocks = hat.reshape(4, 2, 2)
    return {"S": S, "R": R, "Lh": blocks[0], "Dh": blocks[1], "Uh": blocks[2], "Dh_first": blocks[3],
            "window": w.value}


def ctri_penta_block_pcr(P: int, n: int, bands, cyclic=True, max_stages=16):
    """Host-only: 2x2-block PCR tables of the pentadiagonal reduced system (alpha, gamma, fold)."""
    a = np.zeros(max_stages * P * 4)
    g = np.zeros(max_stages * P * 4)
    f = np.zeros(P * 4)
    q = ctypes.c_int()
    dp = ctypes.POINTER(ctypes.c_double)
    _check(load().ctri_penta_block_pcr(int(P), int(bool(cyclic)), int(n), _dbl5(bands), int(max_stages),
                                       a.ctypes.data_as(dp), g.ctypes.data_as(dp), f.ctypes.data_as(dp),
                                       ctypes.byref(q)), "ctri_penta_block_pcr")
    k = q.value
    return a[:k * P * 4].reshape(k, P, 2, 2), g[:k * P * 4].reshape(k, P, 2, 2), f.reshape(P, 2, 2)


def ctri_penta_reduced_schedule_apply(P: int, n: int, bands, bhat, cyclic=True):
    """Host-only: the pentadiagonal reduced system's step schedule (block PCR, or block detach /
    PCR / fold / reattach) applied to bhat [P, 2]; returns (x~ [P, 2], steps, detach stages,
    detached rows)."""
    b = np.ascontiguousarray(bhat, dtype=np.float64).reshape(2 * P)
    x = np.zeros(2 * P)
    k, ds, dr = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    dp = ctypes.POINTER(ctypes.c_double)
    _check(load().ctri_penta_reduced_schedule_apply(int(P), int(bool(cyclic)), int(n), _dbl5(bands),
                                                    b.ctypes.data_as(dp), x.ctypes.data_as(dp),
                                                    ctypes.byref(k), ctypes.byref(ds), ctypes.byref(dr)),
           "ctri_penta_reduced_schedule_apply")
    return x.reshape(P, 2), k.value, ds.value, dr.value


def ctri_solve(plan: int, b, x, stream=None):
    _check(load().ctri_solve(plan, _ptr(b), _ptr(x), _stream_ptr(stream)), "ctri_solve")


def ctri_solve_loopback(plans, bs, xs, stream=None):
    n = len(plans)
    hp = (ctypes.c_void_p * n)(*plans)
    bp = (ctypes.c_void_p * n)(*[_ptr(b) for b in bs])
    xp = (ctypes.c_void_p * n)(*[_ptr(x) for x in xs])
    _check(load().ctri_solve_loopback(hp, n, bp, xp, _stream_ptr(stream)), "ctri_solve_loopback")


def ctri_solve_host(plan: int, b_host, x_host, stream=None):
    _check(load().ctri_solve_host(plan, _ptr(b_host), _ptr(x_host), _stream_ptr(stream)),
           "ctri_solve_host")


def _opt(v, none):
    return none if v is None else float(v)


def ctri_deriv(plan: int, f, df, a=None, bc=None, h=None, stream=None):
    """a, bc, h = None: the library's defaults (Lele's a = 14/9, bc = 1/9; h = 2 pi / N)."""
    _check(load().ctri_deriv(plan, _ptr(f), _ptr(df), _opt(a, float("nan")), _opt(bc, float("nan")),
                             _opt(h, 0.0), _stream_ptr(stream)), "ctri_deriv")


def ctri_deriv_loopback(plans, fs, dfs, a=None, bc=None, h=None, stream=None):
    n = len(plans)
    hp = (ctypes.c_void_p * n)(*plans)
    fp = (ctypes.c_void_p * n)(*[_ptr(f) for f in fs])
    dp = (ctypes.c_void_p * n)(*[_ptr(d) for d in dfs])
    _check(load().ctri_deriv_loopback(hp, n, fp, dp, _opt(a, float("nan")), _opt(bc, float("nan")),
                                      _opt(h, 0.0), _stream_ptr(stream)), "ctri_deriv_loopback")


def _coef5(coef):
    c = (ctypes.c_double * 5)(*[float(v) for v in coef])
    if len(coef) != 5:
        raise ValueError("coef must hold 5 values (offsets -2..2)")
    return ctypes.cast(c, ctypes.POINTER(ctypes.c_double)), c


def ctri_compact_apply(plan: int, coef, f, out, stream=None):
    cp, _keep = _coef5(coef)
    _check(load().ctri_compact_apply(plan, cp, _ptr(f), _ptr(out), _stream_ptr(stream)),
           "ctri_compact_apply")


def ctri_compact_apply_loopback(plans, coef, fs, outs, stream=None):
    n = len(plans)
    hp = (ctypes.c_void_p * n)(*plans)
    fp = (ctypes.c_void_p * n)(*[_ptr(f) for f in fs])
    op = (ctypes.c_void_p * n)(*[_ptr(o) for o in outs])
    cp, _keep = _coef5(coef)
    _check(load().ctri_compact_apply_loopback(hp, n, cp, fp, op, _stream_ptr(stream)),
           "ctri_compact_apply_loopback")


CTRI_SCHEME_COLLOCATED_D1 = 0
CTRI_SCHEME_STAGGERED_D1 = 1
CTRI_SCHEME_STAGGERED_I = 2


def ctri_scheme_coef(scheme: int, delta: float = 1.0):
    """(coef[5], bands[3]) of a compact scheme of the paper, computed by the library."""
    c = (ctypes.c_double * 5)()
    bd = (ctypes.c_double * 3)()
    _check(load().ctri_scheme_coef(int(scheme), float(delta), c, bd), "ctri_scheme_coef")
    return tuple(c), tuple(bd)


def staggered_deriv_coef(delta: float):
    return ctri_scheme_coef(CTRI_SCHEME_STAGGERED_D1, delta)[0]


def staggered_interp_coef():
    return ctri_scheme_coef(CTRI_SCHEME_STAGGERED_I)[0]


def staggered_deriv_bands():
    return ctri_scheme_coef(CTRI_SCHEME_STAGGERED_D1)[1]


def staggered_interp_bands():
    return ctri_scheme_coef(CTRI_SCHEME_STAGGERED_I)[1]


def ctri_get_stats(plan: int) -> dict:
    s = ctri_stats()
    _check(load().ctri_get_stats(plan, ctypes.byref(s)), "ctri_get_stats")
    return s.as_dict()


def ctri_plan_destroy(plan: int):
    _check(load().ctri_plan_destroy(plan), "ctri_plan_destroy")


def ctri_factor_query(n: int, bands=(1 / 3, 1.0, 1 / 3)):
    """Host-only: S, R (n-1 each), (L^, D^, U^) and the back-substitution window W."""
    S = np.zeros(max(1, n - 1))
    R = np.zeros(max(1, n - 1))
    hat = np.zeros(3)
    w = ctypes.c_int()
    dp = ctypes.POINTER(ctypes.c_double)
    _check(load().ctri_factor_query(int(n), _dbl3(bands), S.ctypes.data_as(dp), R.ctypes.data_as(dp),
                                    hat.ctypes.data_as(dp), ctypes.byref(w)), "ctri_factor_query")
    return S, R, tuple(hat), w.value


def ctri_pcr_coefficients(L, D, U, cyclic=True):
    """Host-only: PCR multipliers alpha/gamma [stages][P] and the final inverse diagonal."""
    L = np.ascontiguousarray(L, dtype=np.float64)
    D = np.ascontiguousarray(D, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64)
    P = len(D)
    a = np.zeros(CTRI_MAX_STAGES * P)
    g = np.zeros(CTRI_MAX_STAGES * P)
    inv = np.zeros(P)
    stages = ctypes.c_int()
    dp = ctypes.POINTER(ctypes.c_double)
    _check(load().ctri_pcr_coefficients(P, int(bool(cyclic)), L.ctypes.data_as(dp),
                                        D.ctypes.data_as(dp), U.ctypes.data_as(dp),
                                        a.ctypes.data_as(dp), g.ctypes.data_as(dp),
                                        inv.ctypes.data_as(dp), ctypes.byref(stages)),
           "ctri_pcr_coefficients")
    q = stages.value
    return a[: q * P].reshape(q, P), g[: q * P].reshape(q, P), inv


def ctri_reduced_schedule(L, D, U, cyclic=True, max_steps=32):
    """Host-only: the reduced-system step schedule (see include/ctri.h).  Returns
    (kinds[nsteps], w[nsteps, P], src[nsteps, P, 2], c[nsteps, P, 2], counts dict)."""
    L = np.ascontiguousarray(L, dtype=np.float64)
    D = np.ascontiguousarray(D, dtype=np.float64)
    U = np.ascontiguousarray(U, dtype=np.float64)
    P = len(D)
    ip = ctypes.POINTER(ctypes.c_int)
    dp = ctypes.POINTER(ctypes.c_double)
    kinds = np.zeros(max_steps, dtype=np.int32)
    w = np.zeros(max_steps * P)
    src = np.zeros(2 * max_steps * P, dtype=np.int32)
    c = np.zeros(2 * max_steps * P)
    counts = np.zeros(3, dtype=np.int32)
    ns = ctypes.c_int()
    _check(load().ctri_reduced_schedule(P, int(bool(cyclic)), L.ctypes.data_as(dp), D.ctypes.data_as(dp),
                                        U.ctypes.data_as(dp), max_steps, ctypes.byref(ns),
                                        kinds.ctypes.data_as(ip), w.ctypes.data_as(dp),
                                        src.ctypes.data_as(ip), c.ctypes.data_as(dp),
                                        counts.ctypes.data_as(ip)), "ctri_reduced_schedule")
    n = ns.value
    return (kinds[:n].copy(), w[: n * P].reshape(n, P), src[: 2 * n * P].reshape(n, P, 2),
            c[: 2 * n * P].reshape(n, P, 2),
            {"pcr_stages": int(counts[0]), "detach_stages": int(counts[1]),
             "detached_rows": int(counts[2])})


# ---------------------------------------------------------------- conveniences
def ctri_reduced_inverse(L, D, U, cyclic=True):
    """Host-only: dense A^{-1} of the reduced system (all-gather table), P x P."""
    L, D, U = (np.ascontiguousarray(v, dtype=np.float64) for v in (L, D, U))
    P_ = len(D)
    out = np.zeros((P_, P_))
    dp = ctypes.POINTER(ctypes.c_double)
    _check(load().ctri_reduced_inverse(P_, int(bool(cyclic)), L.ctypes.data_as(dp), D.ctypes.data_as(dp),
                                       U.ctypes.data_as(dp), out.ctypes.data_as(dp)),
           "ctri_reduced_inverse")
    return out


def local_shape(global_dims, solve_dim, nparts):
    s = list(global_dims)
    s[solve_dim] //= nparts
    return tuple(s)


class Plan:
    """One rank's plan.  With nparts > 1 pass the shared NCCL ``unique_id``
    (see :func:`paper_2101_02286_b200.dist.plan_from_process_group`)."""

    def __init__(self, global_dims, solve_dim=0, nparts=1, rank=0, bands=(1 / 3, 1.0, 1 / 3),
                 cyclic=True, unique_id=None, flags=0, stream=None):
        self.global_dims = tuple(int(d) for d in global_dims)
        self.solve_dim = int(solve_dim)
        self.nparts = int(nparts)
        self.rank = int(rank)
        create = ctri_plan_create_penta if len(bands) == 5 else ctri_plan_create
        self.handle = create(global_dims, solve_dim, nparts, rank, bands, cyclic, unique_id, flags, stream)

    @property
    def local_shape(self):
        return local_shape(self.global_dims, self.solve_dim, self.nparts)

    @property
    def local_numel(self):
        return int(np.prod(self.local_shape))

    def solve(self, b, x=None, stream=None):
        if x is None:
            x = b
        n = self.local_numel
        ctri_solve(self.handle, _dev(b, n, "b"), _dev(x, n, "x"), stream)
        return x

    def solve_host(self, b_host, x_host, stream=None):
        n = self.local_numel
        ctri_solve_host(self.handle, _host(b_host, n, "b_host"), _host(x_host, n, "x_host"), stream)
        return x_host

    def deriv(self, f, df, a=None, bc=None, h=None, stream=None):
        n = self.local_numel
        ctri_deriv(self.handle, _dev(f, n, "f"), _dev(df, n, "df"), a, bc, h, stream)
        return df

    def compact_apply(self, coef, f, out, stream=None):
        n = self.local_numel
        ctri_compact_apply(self.handle, coef, _dev(f, n, "f"), _dev(out, n, "out"), stream)
        return out

    def stats(self) -> dict:
        return ctri_get_stats(self.handle)

    def close(self):
        if self.handle:
            ctri_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class LoopbackGroup:
    """TEST-ONLY: nparts ranks on one device, exchanges as device copies."""

    def __init__(self, global_dims, solve_dim, nparts, bands=(1 / 3, 1.0, 1 / 3), cyclic=True,
                 flags=0, stream=None):
        self.global_dims = tuple(int(d) for d in global_dims)
        self.solve_dim = int(solve_dim)
        self.nparts = int(nparts)
        create = ctri_plan_create_penta_loopback if len(bands) == 5 else ctri_plan_create_loopback
        self.handles = create(global_dims, solve_dim, nparts, bands, cyclic, flags, stream)

    @property
    def local_shape(self):
        return local_shape(self.global_dims, self.solve_dim, self.nparts)

    def _chk(self, ts, what):
        if len(ts) != self.nparts:
            raise ValueError(f"{what}: {len(ts)} slabs for {self.nparts} ranks")
        n = int(np.prod(self.local_shape))
        return [_dev(t, n, f"{what}[{r}]") for r, t in enumerate(ts)]

    def solve(self, bs, xs, stream=None):
        ctri_solve_loopback(self.handles, self._chk(bs, "b"), self._chk(xs, "x"), stream)

    def deriv(self, fs, dfs, a=None, bc=None, h=None, stream=None):
        ctri_deriv_loopback(self.handles, self._chk(fs, "f"), self._chk(dfs, "df"), a, bc, h, stream)

    def compact_apply(self, coef, fs, outs, stream=None):
        ctri_compact_apply_loopback(self.handles, coef, self._chk(fs, "f"), self._chk(outs, "out"), stream)

    def stats(self, rank=0):
        return ctri_get_stats(self.handles[rank])

    def close(self):
        for h in self.handles or []:
            ctri_plan_destroy(h)
        self.handles = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
