// kernels.cu -- sm_100a kernels of the batched cyclic tridiagonal solve.
//
// Steps of the paper's method (PAPER.md Sec. "Parallel linear solver"):
//   (a1) local solve y_i = D_i^{-1} b_i                      k_tile (tile.cu) / k_local_generic
//   (a2) reduced RHS b^_i = b~_i - l y_{i-1}[last] - u y_i[0]  k_bhat       (Eq. bi_hat)
//   (a3) one cyclic PCR stage on A^ x~ = b^                  k_pcr_stage
//   (a4) x_i = y_i - S_i x~_i - R_i x~_{i+1}                 k_backsub     (Eq. xi_app)
//   (a0) compact-derivative RHS stencil                      k_stencil
//
// The hot kernel, k_tile, lives in tile.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace ctri {

static inline unsigned blocks_for(int64_t m, int bs) { return (unsigned)((m + bs - 1) / bs); }


// ------------------------------------------------------------------------------------------
// (a1) generic column-serial local solve: one thread per batch column, any n >= 3, any layout.
// mode 0 (nparts = 1): complete cyclic solve; mode 1: y = D_i^{-1} b_i into x + planes.
// ------------------------------------------------------------------------------------------
__global__ void k_local_generic(const double* b, double* x, int64_t outer, int64_t n,
                                int64_t inner, const double* __restrict__ cp,
                                const double* __restrict__ inv_den, double l, double u, int mode,
                                const double* __restrict__ S, const double* __restrict__ R,
                                double inv_closure, int cyc, double* yf, double* yl, double* bt) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= outer * inner) return;
  const int64_t o = t / inner, c = t - o * inner;
  const double* bc = b + o * n * inner + c;
  double* xc = x + o * n * inner + c;
  const int64_t st = inner;
  const double btv = bc[0];
  // Thomas forward over interior rows 1..n-1 (Eq. yi)
  double g = bc[st] * inv_den[0];
  xc[st] = g;
  for (int64_t r = 2; r < n; ++r) {
    g = (bc[r * st] - l * g) * inv_den[r - 1];
    xc[r * st] = g;
  }
  const double ylast = g;
  double y = g;
  for (int64_t r = n - 2; r >= 1; --r) {
    y = xc[r * st] - cp[r - 1] * y;
    xc[r * st] = y;
  }
  const double yfirst = y;
  if (mode == 0) {
    // p = 1: the reduced system is the 1x1 closure (L^+D^+U^) x~ = b^
    // (acyclic p = 1: no wrap coupling, L~ = 0 and U = 0, so no l-term and no R-term)
    const double bh = btv - (cyc ? l * ylast : 0.0) - u * yfirst;
    const double xt = bh * inv_closure;
    const double xr = cyc ? xt : 0.0;
    xc[0] = xt;
    for (int64_t r = 1; r < n; ++r) xc[r * st] = xc[r * st] - S[r - 1] * xt - R[r - 1] * xr;
  } else {
    xc[0] = btv;
    yf[t] = yfirst;
    yl[t] = ylast;
    bt[t] = btv;
  }
}

// (a2) b^_i = b~_i - l y_{i-1}[last] - u y_i[first]   (Eq. bi_hat)
__global__ void k_bhat(const double* __restrict__ bt, const double* __restrict__ yl_prev,
                       const double* __restrict__ yf, double* __restrict__ bh, int64_t m, double l,
                       double u) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < m) bh[j] = bt[j] - l * yl_prev[j] - u * yf[j];
}

// (a3) one PCR stage: b^_i <- b^_i - alpha b^_{i-s} - gamma b^_{i+s}; last stage scales by inv.
__global__ void k_pcr_stage(double* bh, const double* __restrict__ rm,
                            const double* __restrict__ rp, int64_t m, double a, double g,
                            int last, double inv, double* __restrict__ xt) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const double v = bh[j] - a * rm[j] - g * rp[j];
  if (last) xt[j] = v * inv;
  else bh[j] = v;
}

// (a4) x_i = y_i - S_i x~_i - R_i x~_{i+1} on rows {0} U window (or all rows); row 0 := x~_i.
__global__ void k_backsub(double* x, int64_t outer, int64_t n, int64_t inner,
                          const double* __restrict__ S, const double* __restrict__ R,
                          const double* __restrict__ xt, const double* __restrict__ xt_next,
                          int64_t W, int full) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t m = outer * inner;
  if (j >= m) return;
  const int64_t ry = blockIdx.y;  // 0 .. rows-1
  int64_t r;
  if (full) {
    r = ry;  // 0..n-1
  } else {
    // rows: 0, 1..W, n-W..n-1
    if (ry == 0) r = 0;
    else if (ry <= W) r = ry;
    else r = n - W + (ry - W - 1);
  }
  const int64_t o = j / inner, c = j - o * inner;
  double* p = x + (o * n + r) * inner + c;
  const double a = xt[j];
  if (r == 0) {
    *p = a;
  } else {
    *p = *p - S[r - 1] * a - R[r - 1] * xt_next[j];
  }
}

// (a4) windowed back-substitution x = y - S x~_s - R x~_{s+1} (Eq. xi_app; window R15)
// of every (virtual) slab s, after the reduced kernel stored x~_s in row 0 of slab s.
// x~_{s+1} is row 0 of slab s+1, or for the last slab: next[j] (the right neighbour's x~, p > 1),
// else row 0 of slab 0 (p == 1 cyclic), else 0 (acyclic end).  A separate high-occupancy
// pass: HBM-bound read-modify-write of 2W rows per slab, 8 independent rows in flight per thread.
struct WindowArgs {
  double* x;
  const double *S, *R, *next;
  int64_t outer, nv, inner, W, rows;
  int vp, full, wrap;
  int pdl;  // launched with programmatic stream serialization: wait for the previous kernel
};
constexpr int kWinRows = 8, kWinBatches = 3;

__device__ __forceinline__ int64_t window_row(const WindowArgs& A, int64_t ry) {
  return A.full ? ry + 1 : (ry < A.W ? ry + 1 : A.nv - 2 * A.W + ry);
}

// strided axis (inner > 1): block = 256 consecutive columns x kWinRows rows of one slab
__global__ void __launch_bounds__(256) k_window(const WindowArgs A) {
  if (A.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");  // launched early (PDL)
  const int64_t j = blockIdx.x * 256ll + threadIdx.x;
  const int64_t m = A.outer * A.inner;
  if (j >= m) return;
  const int s = blockIdx.z;
  const int64_t o = j / A.inner, c = j - o * A.inner;
  const int64_t sl = A.nv * A.inner;  // one slab
  double* xs = A.x + (o * A.vp + s) * sl + c;
  const double xa = xs[0];
  double xn = 0.0;
  if (s + 1 < A.vp) xn = xs[sl];
  else if (A.next) xn = A.next[j];
  else if (A.wrap) xn = A.x[o * A.vp * sl + c];
  // kWinBatches batches of kWinRows rows per thread: the grid stays within about one wave
  for (int bt = 0; bt < kWinBatches; ++bt) {
    const int64_t r0 = ((int64_t)blockIdx.y * kWinBatches + bt) * kWinRows;
    if (r0 >= A.rows) break;
    double v[kWinRows];
#pragma unroll
    for (int u = 0; u < kWinRows; ++u)
      if (r0 + u < A.rows) v[u] = xs[window_row(A, r0 + u) * A.inner];
#pragma unroll
    for (int u = 0; u < kWinRows; ++u)
      if (r0 + u < A.rows) {
        const int64_t r = window_row(A, r0 + u);
        dev::st_global_cs(xs + r * A.inner, v[u] - __ldg(A.S + r - 1) * xa - __ldg(A.R + r - 1) * xn);
      }
  }
}

// strided axis with an even row length (the usual case): a thread owns a PAIR of adjacent
// columns (16-byte loads and stores) and kWinPairRows consecutive window rows of one slab, all
// loads in flight before the first store; rows walk by pointer increments, so the per-element
// work is one load, one store and four DFMA per pair (the per-element 64-bit index arithmetic of
// k_window made that kernel issue-bound: ncu cfg3 slab, 60% issue slots busy at 2.5 TB/s)
constexpr int kWinPairRows = 8;
__global__ void __launch_bounds__(256) k_window_pairs(const WindowArgs A) {
  if (A.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");  // launched early (PDL)
  const int64_t j = 2 * (blockIdx.x * 256ll + threadIdx.x);        // first column of the pair
  const int64_t m = A.outer * A.inner;
  if (j >= m) return;
  const int s = blockIdx.z;
  const int64_t o = j / A.inner, c = j - o * A.inner;
  const int64_t sl = A.nv * A.inner;  // one slab
  double* xs = A.x + (o * A.vp + s) * sl + c;
  const double2 xa = *reinterpret_cast<const double2*>(xs);
  double2 xn = make_double2(0.0, 0.0);
  if (s + 1 < A.vp) xn = *reinterpret_cast<const double2*>(xs + sl);
  else if (A.next) xn = *reinterpret_cast<const double2*>(A.next + j);
  else if (A.wrap) xn = *reinterpret_cast<const double2*>(A.x + o * A.vp * sl + c);
  const int r0 = blockIdx.y * kWinPairRows;  // first window row index of this thread
  double2 v[kWinPairRows];
  double* pr[kWinPairRows];
#pragma unroll
  for (int u = 0; u < kWinPairRows; ++u) {
    const int ry = r0 + u;
    const int64_t r = window_row(A, ry);
    pr[u] = xs + r * A.inner;
    if (ry < A.rows) v[u] = *reinterpret_cast<const double2*>(pr[u]);
  }
#pragma unroll
  for (int u = 0; u < kWinPairRows; ++u) {
    const int ry = r0 + u;
    if (ry < A.rows) {
      const int64_t r = window_row(A, ry);
      const double sv = __ldg(A.S + r - 1), rv = __ldg(A.R + r - 1);
      dev::st_global_cs_v2(pr[u], v[u].x - sv * xa.x - rv * xn.x, v[u].y - sv * xa.y - rv * xn.y);
    }
  }
}

// contiguous axis (inner == 1): one warp per column, lanes along the (contiguous) rows
__global__ void __launch_bounds__(256) k_window_contig(const WindowArgs A) {
  const int64_t w = blockIdx.x * 8ll + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= A.outer * A.vp) return;
  const int64_t o = w / A.vp;
  const int s = (int)(w - o * A.vp);
  double* xs = A.x + w * A.nv;
  const double xa = xs[0];
  double xn = 0.0;
  if (s + 1 < A.vp) xn = xs[A.nv];
  else if (A.next) xn = A.next[o];
  else if (A.wrap) xn = A.x[o * A.vp * A.nv];
  for (int64_t r0 = 0; r0 < A.rows; r0 += 32 * 4) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t ry = r0 + u * 32 + lane;
      if (ry < A.rows) v[u] = xs[window_row(A, ry)];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t ry = r0 + u * 32 + lane;
      if (ry < A.rows) {
        const int64_t r = window_row(A, ry);
        xs[r] = v[u] - __ldg(A.S + r - 1) * xa - __ldg(A.R + r - 1) * xn;
      }
    }
  }
}

// contiguous axis, window of at most 96 rows per partition (the usual case): persistent warps
// walk the (column, partition) units; a lane's rows, their offsets and their S, R are the same
// for every unit, so they are computed once, and two units are loaded before either is
// corrected (the per-unit version spent its issue slots on index arithmetic: ncu cfg4 index 2,
// 56% issue-busy at 3.2 TB/s)
constexpr int kWinUnitRows = 3;  // rows per lane: 96 >= the window
constexpr int kWinUnroll = 4;    // units per warp in flight
__global__ void __launch_bounds__(256) k_window_contig_units(const WindowArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t units = A.outer * A.vp;
  const int64_t nw = (int64_t)gridDim.x * 8;
  const int vsh = __ffs(A.vp) - 1;  // vp is a power of two
  int64_t roff[kWinUnitRows];
  double sv[kWinUnitRows], rv[kWinUnitRows];
  bool act[kWinUnitRows];
#pragma unroll
  for (int u = 0; u < kWinUnitRows; ++u) {
    const int64_t ry = lane + 32 * u;
    act[u] = ry < A.rows;
    roff[u] = act[u] ? window_row(A, ry) : 0;
    sv[u] = act[u] ? __ldg(A.S + roff[u] - 1) : 0.0;
    rv[u] = act[u] ? __ldg(A.R + roff[u] - 1) : 0.0;
  }
  for (int64_t w0 = blockIdx.x * 8ll + (threadIdx.x >> 5); w0 < units; w0 += kWinUnroll * nw) {
    double v[kWinUnroll][kWinUnitRows], xa[kWinUnroll], xn[kWinUnroll];
#pragma unroll
    for (int q = 0; q < kWinUnroll; ++q) {
      const int64_t w = w0 + q * nw;
      xa[q] = xn[q] = 0.0;
      if (w >= units) continue;
      const int64_t o = w >> vsh;
      const int sp = (int)(w - (o << vsh));
      const double* xs = A.x + w * A.nv;
      xa[q] = xs[0];
      if (sp + 1 < A.vp) xn[q] = xs[A.nv];
      else if (A.next) xn[q] = A.next[o];
      else if (A.wrap) xn[q] = A.x[(o << vsh) * A.nv];
#pragma unroll
      for (int u = 0; u < kWinUnitRows; ++u)
        if (act[u]) v[q][u] = xs[roff[u]];
    }
#pragma unroll
    for (int q = 0; q < kWinUnroll; ++q) {
      const int64_t w = w0 + q * nw;
      if (w >= units) continue;
      double* xs = A.x + w * A.nv;
#pragma unroll
      for (int u = 0; u < kWinUnitRows; ++u)
        if (act[u]) xs[roff[u]] = v[q][u] - sv[u] * xa[q] - rv[u] * xn[q];
    }
  }
}

cudaError_t launch_window(const Plan& P, double* x, const double* next, cudaStream_t s) {
  WindowArgs A;
  A.x = x;
  A.S = P.d_S;
  A.R = P.d_R;
  A.next = next;
  A.outer = P.lay.outer;
  A.nv = P.lay.n / P.rvp;  // the reduced system's partitions (virtual rows, or whole slabs)
  A.inner = P.lay.inner;
  A.W = P.window;
  A.full = ((P.flags & CTRI_FLAG_FULL_BACKSUB) || (2 * P.window >= A.nv - 1)) ? 1 : 0;
  A.rows = A.full ? A.nv - 1 : 2 * A.W;
  A.vp = P.rvp;
  A.wrap = (P.p == 1 && P.cyclic) ? 1 : 0;
  A.pdl = 0;
  if (A.rows <= 0) return cudaSuccess;
  if (A.inner == 1) {
    const int64_t warps = A.outer * A.vp;
    if (A.rows <= 32 * kWinUnitRows && (A.vp & (A.vp - 1)) == 0) {
      // persistent: 6 blocks of 8 warps per SM, every warp several units
      const int64_t blocks = std::min<int64_t>((warps + 8 * kWinUnroll - 1) / (8 * kWinUnroll), (int64_t)P.num_sms * 6);
      k_window_contig_units<<<(unsigned)std::max<int64_t>(blocks, 1), 256, 0, s>>>(A);
    } else {
      k_window_contig<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(A);
    }
  } else {
    const int64_t m = P.lay.m();
    const bool pairs = (A.inner % 2) == 0;  // (ncu, cold: cfg3 slab 18.1 -> 16.7 us, cfg2 N=2 62 -> 57 us)
    const int64_t rpb = pairs ? (int64_t)kWinPairRows : (int64_t)kWinRows * kWinBatches;
    const int64_t cpb = pairs ? 512 : 256;  // columns per block
    dim3 grid((unsigned)((m + cpb - 1) / cpb), (unsigned)((A.rows + rpb - 1) / rpb), (unsigned)A.vp);
    // after the P2P kernel (nparts > 1): programmatic dependent launch, so the window grid is
    // staged while the reduced-phase kernel drains (the kernel waits before touching x)
    A.pdl = (P.p > 1 && !knob_no_pdl()) ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256, 1, 1);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = A.pdl ? 1 : 0;
    return pairs ? cudaLaunchKernelEx(&cfg, k_window_pairs, A) : cudaLaunchKernelEx(&cfg, k_window, A);
  }
  return cudaGetLastError();
}

// (a2)-(a4) for the virtual partitions of one GPU (nparts == 1, vp > 1): per batch column the
// vp-row reduced system (cyclic or acyclic) is formed from the planes (Eq. bi_hat), solved with
// the plan's PCR multipliers (fold R3) and back-substituted on the window rows of
// every virtual slab (Eq. xi_app).  No communication: all partitions live in this slab.
struct LocalRedArgs {
  int vp, q, cyclic, full;
  int64_t outer, nv, inner, W;
  double l, u;
  const double *S, *R, *yf, *yl, *bt;
  double alpha[4 * 8], gamma[4 * 8], inv[8];  // [stage][row], vp <= 8
  int dense;                                  // cyclic, vp not a power of two: x~ = A^-1 b^
  double ainv[8 * 8];                         // [row][row] of the vp-row reduced matrix
};

__device__ __forceinline__ double bh_get(const double (&bh)[8], int v) {
  double r = bh[0];
#pragma unroll
  for (int i = 1; i < 8; ++i)
    if (v == i) r = bh[i];
  return r;
}

__global__ void __launch_bounds__(128) k_reduced_local(const LocalRedArgs A, double* __restrict__ x) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t m = A.outer * A.inner;
  if (j >= m) return;
  const int vp = A.vp;
  const int64_t o = j / A.inner, c = j - o * A.inner;
  double bh[8];
  for (int v = 0; v < 8; ++v) {
    if (v >= vp) break;
    const int64_t pj = (o * vp + v) * A.inner + c;
    const int vl = (v + vp - 1) % vp;
    const double ylp = (A.cyclic || v > 0) ? A.yl[(o * vp + vl) * A.inner + c] : 0.0;
    bh[v] = A.bt[pj] - A.l * ylp - A.u * A.yf[pj];
  }
  if (A.dense) {  // x~_v = sum_w (A^-1)_{vw} b^_w (plan-time inverse; no PCR partner pattern
                  // for a cyclic system of vp rows when vp is not a power of two)
    double xv[8];
    for (int v = 0; v < 8; ++v) {
      if (v >= vp) break;
      double acc = 0.0;
      for (int w = 0; w < 8; ++w)
        if (w < vp) acc += A.ainv[v * vp + w] * bh[w];
      xv[v] = acc;
    }
    for (int v = 0; v < 8; ++v)
      if (v < vp) x[((o * vp + v) * A.nv) * A.inner + c] = xv[v];
    return;
  }
  for (int k = 0; k < A.q; ++k) {
    const int s = 1 << k;
    double nb[8];
    for (int v = 0; v < 8; ++v) {
      if (v >= vp) break;
      int lm = v - s, lp = v + s;
      double vm = 0.0, vpv = 0.0;
      if (A.cyclic) {
        vm = bh[((lm % vp) + vp) % vp];
        vpv = bh[lp % vp];
      } else {
        if (lm >= 0) vm = bh[lm];
        if (lp < vp) vpv = bh[lp];
      }
      nb[v] = bh[v] - A.alpha[k * 8 + v] * vm - A.gamma[k * 8 + v] * vpv;
    }
    for (int v = 0; v < 8; ++v)
      if (v < vp) bh[v] = nb[v];
  }
  for (int v = 0; v < 8; ++v)
    if (v < vp) bh[v] *= A.inv[v];
  // x~ of every virtual slab into its row 0; the window pass (k_window) follows
  for (int v = 0; v < 8; ++v)
    if (v < vp) x[((o * vp + v) * A.nv) * A.inner + c] = bh[v];
}

cudaError_t launch_reduced_local(const Plan& P, double* x, cudaStream_t s) {
  LocalRedArgs A;
  A.vp = P.vp;
  A.q = P.gpcr.stages;
  A.cyclic = P.cyclic;
  A.full = ((P.flags & CTRI_FLAG_FULL_BACKSUB) || (2 * P.window >= P.tlay.n - 1)) ? 1 : 0;
  A.outer = P.lay.outer;
  A.nv = P.tlay.n;
  A.inner = P.lay.inner;
  A.W = P.window;
  A.l = P.bands.l;
  A.u = P.bands.u;
  A.S = P.d_S;
  A.R = P.d_R;
  A.yf = P.yf;
  A.yl = P.yl;
  A.bt = P.bt;
  for (int i = 0; i < 32; ++i) A.alpha[i] = A.gamma[i] = 0.0;
  for (int i = 0; i < 64; ++i) A.ainv[i] = 0.0;
  A.dense = (P.cyclic && (P.vp & (P.vp - 1)) != 0) ? 1 : 0;
  if (A.dense) {  // (the plan holds A^-1 of the vp-row system; no PCR tables)
    if (P.ainv.size() != (size_t)P.vp * P.vp) return cudaErrorInvalidValue;
    A.q = 0;
    for (int i = 0; i < P.vp * P.vp; ++i) A.ainv[i] = P.ainv[i];
  }
  for (int kk = 0; kk < A.q && kk < 4; ++kk)
    for (int v = 0; v < P.vp; ++v) {
      A.alpha[kk * 8 + v] = P.gpcr.alpha[(size_t)kk * P.vp + v];
      A.gamma[kk * 8 + v] = P.gpcr.gamma[(size_t)kk * P.vp + v];
    }
  for (int v = 0; v < 8; ++v) A.inv[v] = (v < P.vp && !A.dense) ? P.gpcr.inv[v] : 0.0;
  const int64_t m = P.lay.m();
  k_reduced_local<<<blocks_for(m, 128), 128, 0, s>>>(A, x);
  return cudaGetLastError();
}

// (a0) pack the two first / two last planes of f into contiguous send buffers (halo exchange).
__global__ void k_pack_halo(const double* __restrict__ f, int64_t outer, int64_t n, int64_t inner,
                            double* __restrict__ send_lo, double* __restrict__ send_hi) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t m = outer * inner;
  if (j >= m) return;
  const int64_t o = j / inner, c = j - o * inner;
  const double* fc = f + o * n * inner + c;
  send_lo[j] = fc[0];
  send_lo[m + j] = fc[inner];
  send_hi[j] = fc[(n - 2) * inner];
  send_hi[m + j] = fc[(n - 1) * inner];
}

// (a0) rhs_r = a (f_{r+1}-f_{r-1})/(2h) + bc (f_{r+2}-f_{r-2})/(4h).
// Rows outside the slab come from halo_lo (rows n-2, n-1 of rank i-1) / halo_hi (rows 0, 1 of
// rank i+1); with nparts = 1 the wrap stays inside the slab.
__global__ void k_stencil(const double* __restrict__ f, double* __restrict__ rhs, int64_t outer,
                          int64_t n, int64_t inner, const double* __restrict__ halo_lo,
                          const double* __restrict__ halo_hi, int wrap, const Stencil5 st) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t m = outer * inner;
  if (j >= m) return;
  const int64_t r = blockIdx.y;
  const int64_t o = j / inner, c = j - o * inner;
  const double* fc = f + o * n * inner + c;
  auto at = [&](int64_t rr) -> double {
    if (rr >= 0 && rr < n) return fc[rr * inner];
    if (wrap) return fc[((rr % n + n) % n) * inner];
    if (rr < 0) return halo_lo[(rr + 2) * m + j];
    return halo_hi[(rr - n) * m + j];
  };
  const double v = apply_stencil5(st, at(r - 2), at(r - 1), at(r), at(r + 1), at(r + 2));
  rhs[(o * n + r) * inner + c] = v;
}

// ------------------------------------------------------------------------------------------
// host launchers
// ------------------------------------------------------------------------------------------

cudaError_t launch_local_generic(const Plan& P, const double* b, double* x, cudaStream_t s) {
  const Layout& L = P.tlay;
  const int64_t m = L.m();
  const int bs = 128;
  k_local_generic<<<blocks_for(m, bs), bs, 0, s>>>(
      b, x, L.outer, L.n, L.inner, P.d_cp, P.d_inv_den, P.bands.l, P.bands.u,
      (P.p == 1 && P.vp == 1) ? 0 : 1, P.d_S, P.d_R, P.inv_closure, P.cyclic, P.yf, P.yl, P.bt);
  return cudaGetLastError();
}

cudaError_t launch_bhat(const Plan& P, cudaStream_t s) {
  const int64_t m = P.lay.m();
  k_bhat<<<blocks_for(m, 256), 256, 0, s>>>(P.bt, P.yl_prev, P.yf, P.bh, m, P.bands.l, P.bands.u);
  return cudaGetLastError();
}

cudaError_t launch_pcr_stage(const Plan& P, int k, bool last, cudaStream_t s) {
  const int64_t m = P.lay.m();
  const double a = P.gpcr.alpha[(size_t)k * P.p + P.rank];
  const double g = P.gpcr.gamma[(size_t)k * P.p + P.rank];
  k_pcr_stage<<<blocks_for(m, 256), 256, 0, s>>>(P.bh, P.recv_m, P.recv_p, m, a, g, last ? 1 : 0,
                                                 P.gpcr.inv[P.rank], P.xt);
  return cudaGetLastError();
}

cudaError_t launch_backsub(const Plan& P, double* x, cudaStream_t s) {
  const int64_t m = P.lay.m();
  const bool full = (P.flags & CTRI_FLAG_FULL_BACKSUB) || (2 * P.window >= P.lay.n - 1);
  const int64_t rows = full ? P.lay.n : 1 + 2 * P.window;
  dim3 grid(blocks_for(m, 256), (unsigned)rows);
  k_backsub<<<grid, 256, 0, s>>>(x, P.lay.outer, P.lay.n, P.lay.inner, P.d_S, P.d_R, P.xt,
                                 P.xt_next, P.window, full ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_pack_halo(const Plan& P, const double* f, cudaStream_t s) {
  const int64_t m = P.lay.m();
  k_pack_halo<<<blocks_for(m, 256), 256, 0, s>>>(f, P.lay.outer, P.lay.n, P.lay.inner, P.send_lo,
                                                 P.send_hi);
  return cudaGetLastError();
}

cudaError_t launch_stencil(const Plan& P, const double* f, double* rhs, const Stencil5& st,
                           cudaStream_t s) {
  const int64_t m = P.lay.m();
  dim3 grid(blocks_for(m, 256), (unsigned)P.lay.n);
  k_stencil<<<grid, 256, 0, s>>>(f, rhs, P.lay.outer, P.lay.n, P.lay.inner, P.halo_lo, P.halo_hi,
                                 P.p == 1 ? 1 : 0, st);
  return cudaGetLastError();
}

}  // namespace ctri
