// kernels.cu -- sm_100a kernels of the batched cyclic tridiagonal solve.
//
// Steps of the paper's method (PAPER.md Sec. "Parallel linear solver"):
//   (a1) local solve y_i = D_i^{-1} b_i                      k_tile<K> / k_local_generic
//   (a2) reduced RHS b^_i = b~_i - l y_{i-1}[last] - u y_i[0]  k_bhat       (Eq. bi_hat)
//   (a3) one cyclic PCR stage on A^ x~ = b^                  k_pcr_stage
//   (a4) x_i = y_i - S_i x~_i - R_i x~_{i+1}                 k_backsub     (Eq. xi_app)
//   (a0) compact-derivative RHS stencil                      k_stencil
//
// k_tile<K> is the hot kernel.  It applies the paper's partition method
// hierarchically ON CHIP: a column of n rows is cut into Q = n/K chunks of K
// rows; each thread owns one chunk of one column in registers, solves the
// chunk interior (K-1 rows) serially (the register leaf of the per-partition
// solve, R16), the Q chunk heads form a reduced tridiagonal system
// (Eqs. Li_hat..bi_hat applied at chunk level) solved by PCR in shared memory
// across the CTAs of a thread-block cluster (DSMEM), and every chunk is then
// back-substituted with Eq. xi_app.  Column tiles of kTileCols batch columns
// are streamed HBM -> shared memory by TMA one tile ahead of the compute, so
// HBM sees one read of b and one write of x (16 B per grid point).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include "internal.h"

namespace ctri {

// ------------------------------------------------------------------------------------------
// PTX helpers (sm_90+/sm_100a): shared-memory addressing, mbarrier, TMA, cluster/DSMEM
// ------------------------------------------------------------------------------------------
namespace dev {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ncluster_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_cluster_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_global_cs(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
}  // namespace dev

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
                          const double* __restrict__ halo_hi, int wrap, double ca, double cb) {
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
  const double v = ca * (at(r + 1) - at(r - 1)) + cb * (at(r + 2) - at(r - 2));
  rhs[(o * n + r) * inner + c] = v;
}

// ------------------------------------------------------------------------------------------
// (a1) cluster-tile local solve (hot kernel), strided solve axis (inner >= kTileCols).
// ------------------------------------------------------------------------------------------
template <int K>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_tile(const __grid_constant__ CUtensorMap tmap, const TileArgs A, const TileConsts<K> T) {
  constexpr int C = kTileCols;
  constexpr int NT = kTileThreads;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int rows_cta = A.rows_per_cta;
  const int Q = A.Q;
  const int stages = A.stages;
  double* tile = reinterpret_cast<double*>(smem_raw);
  double* ex_bt = tile + (size_t)rows_cta * C;
  double* ex_yf = ex_bt + NT;
  double* ex_yl = ex_yf + NT;
  double* pb0 = ex_yl + NT;
  double* pb1 = pb0 + NT;
  double* xt_s = pb1 + NT;
  double* s_alpha = xt_s + NT;
  double* s_gamma = s_alpha + (size_t)stages * Q;
  double* s_inv = s_gamma + (size_t)stages * Q;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(s_inv + Q);

  const int tid = threadIdx.x;
  const int j = tid % C;   // column within the tile
  const int cl = tid / C;  // chunk within this CTA
  const int G = A.G;
  const uint32_t g = (G > 1) ? dev::cluster_ctarank() : 0u;
  const int c = (int)g * kTileChunksPerCta + cl;  // chunk index within the column (0..Q-1)
  const int cols_per_owner = C / G;
  const uint32_t owner = (uint32_t)(j / cols_per_owner);
  const int slot = (j % cols_per_owner) * Q + c;
  const int slot_next = (c + 1 < Q) ? slot + 1 : slot + 1 - Q;
  const int oj = tid / Q, oc = tid - (tid / Q) * Q;  // reduced row owned by this thread
  const int prev_row = oj * Q + ((oc - 1) & (Q - 1));

  for (int i = tid; i < stages * Q; i += NT) {
    s_alpha[i] = A.pcr_alpha[i];
    s_gamma[i] = A.pcr_gamma[i];
  }
  for (int i = tid; i < Q; i += NT) s_inv[i] = A.pcr_inv[i];
  const uint32_t bar = dev::smem_u32(mbar);
  if (tid == 0) {
    dev::mbar_init(bar, 1);
    dev::fence_mbar_init();
  }
  __syncthreads();

  const uint32_t ncl = (G > 1) ? dev::ncluster_x() : gridDim.x;
  const int64_t first = (G > 1) ? (int64_t)dev::cluster_id_x() : (int64_t)blockIdx.x;
  const uint32_t tile_bytes = (uint32_t)rows_cta * C * (uint32_t)sizeof(double);
  const int boxr = rows_cta < 256 ? rows_cta : 256;
  const int row0 = (int)g * rows_cta;
  const uint64_t pol = dev::policy_evict_first();

  auto issue = [&](int64_t t) {
    const int o = (int)(t / A.tiles_per_outer);
    const int col0 = (int)(t - (int64_t)o * A.tiles_per_outer) * C;
    dev::fence_proxy_async();
    dev::mbar_expect_tx(bar, tile_bytes);
    for (int r = 0; r < rows_cta; r += boxr)
      dev::tma_load_3d(dev::smem_u32(tile + (size_t)r * C), &tmap, col0, row0 + r, o, bar, pol);
  };

  // remote (owner CTA) addresses of the exchange arrays
  const uint32_t r_bt = (G > 1) ? dev::mapa(dev::smem_u32(ex_bt + slot), owner) : dev::smem_u32(ex_bt + slot);
  const uint32_t r_yf = (G > 1) ? dev::mapa(dev::smem_u32(ex_yf + slot), owner) : dev::smem_u32(ex_yf + slot);
  const uint32_t r_yl = (G > 1) ? dev::mapa(dev::smem_u32(ex_yl + slot), owner) : dev::smem_u32(ex_yl + slot);
  const uint32_t r_xa = (G > 1) ? dev::mapa(dev::smem_u32(xt_s + slot), owner) : dev::smem_u32(xt_s + slot);
  const uint32_t r_xb = (G > 1) ? dev::mapa(dev::smem_u32(xt_s + slot_next), owner) : dev::smem_u32(xt_s + slot_next);

  if (tid == 0 && first < A.num_tiles) issue(first);
  uint32_t phase = 0;
  for (int64_t t = first; t < A.num_tiles; t += ncl) {
    const int64_t o = t / A.tiles_per_outer;
    const int64_t col = (t - o * A.tiles_per_outer) * C + j;
    dev::mbar_wait(bar, phase);
    phase ^= 1u;
    double v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = tile[(cl * K + k) * C + j];
    __syncthreads();  // every thread has its chunk in registers: the buffer is free
    if (tid == 0 && t + ncl < A.num_tiles) issue(t + ncl);

    // ---- chunk interior solve (rows 1..K-1), Thomas with plan-time factors ----
    const double btv = v[0];
    {
      double gg = v[1] * T.inv_den[0];
      v[1] = gg;
#pragma unroll
      for (int k = 2; k < K; ++k) {
        gg = (v[k] - T.l * gg) * T.inv_den[k - 1];
        v[k] = gg;
      }
#pragma unroll
      for (int k = K - 2; k >= 1; --k) v[k] = v[k] - T.cp[k - 1] * v[k + 1];
    }
    // ---- scatter (b~_c, y_c[first], y_c[last]) to the CTA owning this column's reduced rows ----
    if (G > 1) {
      dev::st_cluster_f64(r_bt, btv);
      dev::st_cluster_f64(r_yf, v[1]);
      dev::st_cluster_f64(r_yl, v[K - 1]);
      dev::cluster_sync();
    } else {
      ex_bt[slot] = btv;
      ex_yf[slot] = v[1];
      ex_yl[slot] = v[K - 1];
      __syncthreads();
    }
    // ---- chunk-level reduced system: b^_c (Eq. bi_hat at chunk level) + PCR ----
    {
      const double lt = (A.mode == 2 && oc == 0) ? 0.0 : T.l * ex_yl[prev_row];  // acyclic top
      double bh = ex_bt[tid] - lt - T.u * ex_yf[tid];
      if (A.mode == 1 && oc == 0) bh = 0.0;  // slab row 0 is the GPU interface, not in D_i
      double* cur = pb0;
      double* nxt = pb1;
      for (int k = 0; k < stages; ++k) {
        cur[tid] = bh;
        __syncthreads();
        const int s = 1 << k;
        const double vm = cur[oj * Q + ((oc - s) & (Q - 1))];
        const double vp = cur[oj * Q + ((oc + s) & (Q - 1))];
        bh = bh - s_alpha[k * Q + oc] * vm - s_gamma[k * Q + oc] * vp;
        double* tmp = cur;
        cur = nxt;
        nxt = tmp;
      }
      xt_s[tid] = bh * s_inv[oc];
    }
    double xa, xb;
    if (G > 1) {
      dev::cluster_sync();
      xa = dev::ld_cluster_f64(r_xa);
      xb = dev::ld_cluster_f64(r_xb);
    } else {
      __syncthreads();
      xa = xt_s[slot];
      xb = xt_s[slot_next];
    }
    if (A.mode != 0 && c == Q - 1) xb = 0.0;  // x~_{i+1} outside D_i (mode 1) / acyclic end (2)
    // ---- chunk back-substitution, Eq. xi_app at chunk level ----
    v[0] = (A.mode == 0 || c != 0) ? xa : btv;
#pragma unroll
    for (int k = 1; k < K; ++k) v[k] = v[k] - T.S[k - 1] * xa - T.R[k - 1] * xb;
    if (col < A.lay.inner) {
      double* xp = A.x + (o * A.lay.n + (int64_t)c * K) * A.lay.inner + col;
#pragma unroll
      for (int k = 0; k < K; ++k) dev::st_global_cs(xp + (int64_t)k * A.lay.inner, v[k]);
      if (A.mode == 1) {
        const int64_t pj = o * A.lay.inner + col;
        if (c == 0) {
          A.plane_yf[pj] = v[1];
          A.plane_bt[pj] = btv;
        }
        if (c == Q - 1) A.plane_yl[pj] = v[K - 1];
      }
    }
  }
}

// ------------------------------------------------------------------------------------------
// host launchers
// ------------------------------------------------------------------------------------------
static inline unsigned blocks_for(int64_t m, int bs) { return (unsigned)((m + bs - 1) / bs); }

cudaError_t launch_local_generic(const Plan& P, const double* b, double* x, cudaStream_t s) {
  const int64_t m = P.lay.m();
  const int bs = 128;
  k_local_generic<<<blocks_for(m, bs), bs, 0, s>>>(
      b, x, P.lay.outer, P.lay.n, P.lay.inner, P.d_cp, P.d_inv_den, P.bands.l, P.bands.u,
      P.p == 1 ? 0 : 1, P.d_S, P.d_R, P.inv_closure, P.cyclic, P.yf, P.yl, P.bt);
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

cudaError_t launch_stencil(const Plan& P, const double* f, double* rhs, double a, double bc,
                           double h, cudaStream_t s) {
  const int64_t m = P.lay.m();
  dim3 grid(blocks_for(m, 256), (unsigned)P.lay.n);
  k_stencil<<<grid, 256, 0, s>>>(f, rhs, P.lay.outer, P.lay.n, P.lay.inner, P.halo_lo, P.halo_hi,
                                 P.p == 1 ? 1 : 0, a / (2.0 * h), bc / (4.0 * h));
  return cudaGetLastError();
}

// ---- tile kernel configuration ----
template <int K>
static void fill_consts(const TileConfig& tc, TileConsts<K>* T) {
  const double* c = tc.consts.data();
  T->l = c[0];
  T->u = c[1];
  const int n1 = K - 1;
  for (int k = 0; k < n1; ++k) {
    T->inv_den[k] = c[2 + k];
    T->cp[k] = c[2 + n1 + k];
    T->S[k] = c[2 + 2 * n1 + k];
    T->R[k] = c[2 + 3 * n1 + k];
  }
}

template <int K>
static const void* tile_kernel_ptr() {
  return reinterpret_cast<const void*>(&k_tile<K>);
}

static const void* tile_kernel_for(int K) {
  switch (K) {
    case 2: return tile_kernel_ptr<2>();
    case 4: return tile_kernel_ptr<4>();
    case 8: return tile_kernel_ptr<8>();
    case 16: return tile_kernel_ptr<16>();
    case 32: return tile_kernel_ptr<32>();
  }
  return nullptr;
}

bool tile_configure(Plan& P, std::string* why) {
  TileConfig& tc = P.tile;
  tc = TileConfig();
  const Layout& L = P.lay;
  if (P.flags & CTRI_FLAG_GENERIC_LOCAL) { *why = "forced generic"; return false; }
  if (L.inner < kTileCols || (L.inner % 2) != 0) { *why = "contiguous or narrow solve axis"; return false; }
  if (L.n % kTileChunksPerCta != 0) { *why = "n not a multiple of 32"; return false; }
  if (L.outer > (int64_t)1 << 30 || L.inner > ((int64_t)1 << 31) || L.n > ((int64_t)1 << 31)) {
    *why = "dims too large for TMA coordinates";
    return false;
  }
  const int64_t kg = L.n / kTileChunksPerCta;  // K * G
  int K = 0, G = 0;
  for (int k : {32, 16, 8, 4, 2}) {
    if (kg % k) continue;
    const int64_t g = kg / k;
    if (g >= 1 && g <= kMaxCluster && (g & (g - 1)) == 0) { K = k; G = (int)g; break; }
  }
  if (!K) { *why = "n/32 not expressible as K*G with K<=32, G<=8"; return false; }
  const int Q = kTileChunksPerCta * G;
  // chunk-level tables (Eqs. Si, Ri, Li_hat..Ui_hat on the (K-1)-row chunk interior)
  Partition cp;
  FactorError fe;
  if (!partition_factor(K - 1, P.bands, &cp, &fe)) { *why = "chunk factor: " + fe.detail; return false; }
  tc.consts.clear();
  tc.consts.push_back(P.bands.l);
  tc.consts.push_back(P.bands.u);
  for (int k = 0; k < K - 1; ++k) tc.consts.push_back(cp.th.inv_den[k]);
  for (int k = 0; k < K - 1; ++k) tc.consts.push_back(cp.th.cp[k]);
  for (int k = 0; k < K - 1; ++k) tc.consts.push_back(cp.S[k]);
  for (int k = 0; k < K - 1; ++k) tc.consts.push_back(cp.R[k]);
  std::vector<double> Lr(Q, cp.Lh), Dr(Q, cp.Dh), Ur(Q, cp.Uh);
  const bool cyc = (P.p == 1 && P.cyclic);
  if (P.p > 1) {  // dummy decoupled row 0 (the GPU interface), acyclic over the other heads
    Lr[0] = 0.0; Dr[0] = 1.0; Ur[0] = 0.0;
    Lr[1] = 0.0;
    Ur[Q - 1] = 0.0;
  } else if (!cyc) {  // p = 1 acyclic: head 0 has no chunk above it
    Lr[0] = 0.0;
    Dr[0] = P.bands.d - P.bands.u * cp.S[0];
    Ur[Q - 1] = 0.0;
  }
  if (!pcr_factor(Q, cyc, Lr, Dr, Ur, pivot_threshold(P.bands), &tc.pcr, &fe)) {
    *why = "chunk PCR factor: " + fe.detail;
    return false;
  }
  tc.K = K;
  tc.G = G;
  tc.Q = Q;
  const int rows_cta = kTileChunksPerCta * K;
  tc.smem_bytes = (int)(sizeof(double) * ((size_t)rows_cta * kTileCols + 6 * kTileThreads +
                                          (size_t)(2 * tc.pcr.stages + 1) * Q) + 16);
  const void* fn = tile_kernel_for(K);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, tc.smem_bytes) !=
      cudaSuccess) {
    *why = "cudaFuncSetAttribute(smem) failed";
    cudaGetLastError();
    return false;
  }
  if (G > 1) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(kTileThreads, 1, 1);
  cfg.dynamicSmemBytes = tc.smem_bytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess || nclusters < 1) {
    cudaGetLastError();
    *why = "cluster occupancy query failed";
    return false;
  }
  const int64_t tiles_per_outer = (L.inner + kTileCols - 1) / kTileCols;
  const int64_t num_tiles = L.outer * tiles_per_outer;
  const int64_t ncl = std::min<int64_t>(nclusters, num_tiles);
  tc.grid = (int)(ncl * G);
  tc.ok = true;
  return true;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

template <int K>
static cudaError_t launch_tile_k(const Plan& P, const CUtensorMap& map, const TileArgs& A,
                                 cudaStream_t s) {
  TileConsts<K> T;
  fill_consts<K>(P.tile, &T);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.tile.grid, 1, 1);
  cfg.blockDim = dim3(kTileThreads, 1, 1);
  cfg.dynamicSmemBytes = P.tile.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P.tile.G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_tile<K>, map, A, T);
}

cudaError_t launch_tile(const Plan& P, const double* b, double* x, cudaStream_t s) {
  const TileConfig& tc = P.tile;
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  const Layout& L = P.lay;
  CUtensorMap map;
  cuuint64_t gdim[3] = {(cuuint64_t)L.inner, (cuuint64_t)L.n, (cuuint64_t)L.outer};
  cuuint64_t gstride[2] = {(cuuint64_t)L.inner * 8, (cuuint64_t)(L.n * L.inner * 8)};
  const int rows_cta = kTileChunksPerCta * tc.K;
  cuuint32_t box[3] = {(cuuint32_t)kTileCols, (cuuint32_t)std::min(rows_cta, 256), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(b), gdim, gstride,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  TileArgs A;
  A.b = b;
  A.x = x;
  A.lay = L;
  A.tiles_per_outer = (L.inner + kTileCols - 1) / kTileCols;
  A.num_tiles = L.outer * A.tiles_per_outer;
  A.Q = tc.Q;
  A.G = tc.G;
  A.rows_per_cta = rows_cta;
  A.stages = tc.pcr.stages;
  A.mode = (P.p > 1) ? 1 : (P.cyclic ? 0 : 2);
  A.pcr_alpha = tc.d_pcr;
  A.pcr_gamma = tc.d_pcr + (size_t)tc.pcr.stages * tc.Q;
  A.pcr_inv = tc.d_pcr + (size_t)2 * tc.pcr.stages * tc.Q;
  A.plane_yf = P.yf;
  A.plane_yl = P.yl;
  A.plane_bt = P.bt;
  switch (tc.K) {
    case 2: return launch_tile_k<2>(P, map, A, s);
    case 4: return launch_tile_k<4>(P, map, A, s);
    case 8: return launch_tile_k<8>(P, map, A, s);
    case 16: return launch_tile_k<16>(P, map, A, s);
    case 32: return launch_tile_k<32>(P, map, A, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ctri
