"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic: it only draws random
numbers, builds the structured right-hand sides named in DESIGN.md's input
recipe, and slices global arrays into per-rank slabs.  Both the CUDA path and
the oracle receive the arrays produced here; neither side's results ever flow
back into it.

Shapes follow BASELINE.json ``configs`` (PAPER.md P:5 strong scaling
8192x256^2, P:33 weak scaling 256^3 per GPU, P:5 "dimensions are permuted
correspondingly" for the direction sweep, P:65-67 + SURVEY 8(d) for the
derivative field).
"""
from __future__ import annotations

import math

import numpy as np

SEEDS = {"cfg1": 1, "cfg2": 2, "cfg3": 3, "cfg4": 2, "cfg5": 5, "tests": 6}


def config(name: str, p: int = 1):
    """Global dims and solve dim for a BASELINE.json config (right layout)."""
    if name == "cfg1":
        return (64, 8, 8), 0
    if name == "cfg2":
        return (8192, 256, 256), 0
    if name == "cfg3":
        return (256 * p, 256, 256), 0
    if name == "cfg4_d1":
        return (256, 8192, 256), 1
    if name == "cfg4_d2":
        return (256, 256, 8192), 2
    if name == "cfg5":
        return (1024, 512, 512), 0
    raise KeyError(name)


def uniform(shape, seed: int) -> np.ndarray:
    """b ~ U[-1, 1) i.i.d., numpy PCG64(seed), fp64; generated over the GLOBAL grid
    so the same array is produced whatever the partition count."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-1.0, 1.0, size=tuple(shape))


def fourier_mode(shape, solve_dim: int, k: int) -> np.ndarray:
    """b_j = cos(2*pi*((k*j) mod N)/N) along solve_dim, broadcast over the batch.
    The product k*j is reduced modulo N in integers first."""
    N = shape[solve_dim]
    j = np.arange(N, dtype=np.int64)
    v = np.cos(2.0 * np.pi * ((k * j) % N) / N)
    sh = [1, 1, 1]
    sh[solve_dim] = N
    return np.broadcast_to(v.reshape(sh), shape).copy()


def delta(shape, solve_dim: int, r: int) -> np.ndarray:
    """b = e_r along solve_dim in every column."""
    b = np.zeros(shape)
    idx = [slice(None)] * 3
    idx[solve_dim] = r
    b[tuple(idx)] = 1.0
    return b


CFG5_KAPPAS = (1, 7, 64, 300, 511)


def cfg5_modes(shape, solve_dim: int, seed: int, kappas=CFG5_KAPPAS):
    """Amplitudes A_k(j,k) ~ U[0.5,1.5) and phases phi_k ~ U[0, 2pi) per batch column."""
    rng = np.random.Generator(np.random.PCG64(seed))
    bshape = [s for i, s in enumerate(shape) if i != solve_dim]
    amps = rng.uniform(0.5, 1.5, size=(len(kappas), *bshape))
    phases = rng.uniform(0.0, 2.0 * math.pi, size=(len(kappas), *bshape))
    return amps, phases


def cfg5_field(shape, solve_dim: int, seed: int, kappas=CFG5_KAPPAS) -> np.ndarray:
    """f = sum_k A_k sin(kappa x_i + phi_k), x_i = 2*pi*i/N along solve_dim (P:121 domain)."""
    N = shape[solve_dim]
    amps, phases = cfg5_modes(shape, solve_dim, seed, kappas)
    f = np.zeros(shape)
    for q, kap in enumerate(kappas):
        xi = 2.0 * np.pi * ((kap * np.arange(N, dtype=np.int64)) % N) / N
        sh = [1, 1, 1]
        sh[solve_dim] = N
        xi = xi.reshape(sh)
        A = np.expand_dims(amps[q], solve_dim)
        ph = np.expand_dims(phases[q], solve_dim)
        f += A * np.sin(xi + ph)
    return f


def slab(global_arr: np.ndarray, solve_dim: int, p: int, rank: int) -> np.ndarray:
    """Rank `rank`'s contiguous slab of the global array (equal split along solve_dim)."""
    N = global_arr.shape[solve_dim]
    n = N // p
    idx = [slice(None)] * global_arr.ndim
    idx[solve_dim] = slice(rank * n, (rank + 1) * n)
    return np.ascontiguousarray(global_arr[tuple(idx)])


def assemble(slabs, solve_dim: int) -> np.ndarray:
    return np.concatenate(slabs, axis=solve_dim)


def device_uniform(shape, seed: int, device):
    """Timing-only input drawn on the device (cost is data independent)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    t = torch.empty(tuple(shape), dtype=torch.float64, device=device)
    t.uniform_(-1.0, 1.0, generator=g)
    return t
