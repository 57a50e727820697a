// ptile.cu -- on-chip local solve of a PENTADIAGONAL partition (r = 2), the
// counterpart of k_tile for the paper's w = 5 case ("for a penta-diagonal system (w = 5),
// D~_i is 2x2"; Eqs. Si..xi_app, with 2x2 blocks).
//
// The partition method is applied once more on chip (R16 with r = 2):
//   * a column of the (virtual) slab is cut into Q chunks of K = 32 rows; the first two rows of
//     a chunk are its heads (the chunk-level x~_c, a 2-vector), the other K - 2 its interior;
//   * each thread holds one chunk of one column in registers and solves the pentadiagonal
//     interior with the plan-time LU factors of penta_factor(K - 2) (the register leaf, Eq. yi);
//   * it sends the chunk's planes c_c = b~_c - U~ y_c and w_c = L~ y_c to the CTA that
//     owns the column's head system (st.async into its shared memory, completing on an
//     mbarrier); the owner forms b^_c = c_c - w_{c-1} (Eq. bi_hat) and solves the
//     block-tridiagonal head system by 2x2-block PCR (P:346 in block form, R20): the Q heads of
//     a column are Q lanes of one warp, so every stage is four register shuffles and two 2x2
//     matrix-vector products with plan-time multipliers;
//   * x~_c goes back to the holders of chunks c and c-1 (st.async), and each chunk is
//     back-substituted, x = y - S0 x~_c[0] - S1 x~_c[1] - R0 x~_{c+1}[0] - R1 x~_{c+1}[1]
//     (Eq. xi_app), and stored: 16 B of HBM traffic per point, the column-serial kernel's 32.
// mode 0: one cyclic partition (complete solve); 2: one acyclic partition (complete solve);
// mode 1: y_D = D_i^{-1} b_i of a partition whose rows 0, 1 are its interface (a decoupled dummy
//         head system row) plus the four planes c0 | c1 | w0 | w1 of the partition.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.h"
#include "ptx.cuh"

namespace ctri {

constexpr int kPK = 32, kPC = 32, kPNT = 256, kPCPC = kPNT / kPC;  // rows/chunk, cols, threads
constexpr int kPN = kPK - 2;                                        // interior rows per chunk
constexpr int kPMaxStages = 6, kPMaxQ = 64;                         // Q <= 64 (clusters <= 8)

// chunk-level tables (kernel parameters: constant bank)
struct PTileConsts {
  double lam1[kPN], lam2[kPN], nu1[kPN], imu[kPN];  // interior LU (penta_factor)
  double S0[kPN], S1[kPN], R0[kPN], R1[kPN];        // chunk-level Eqs. Si, Ri (2 columns each)
  double e, l, u, f;
};

__global__ void __launch_bounds__(kPNT, 2)
    k_ptile(const __grid_constant__ CUtensorMap tmap, const PTileArgs A, const PTileConsts T) {
  constexpr int C = kPC, NT = kPNT, K = kPK, CPC = kPCPC, ROWS = CPC * K;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* ring = reinterpret_cast<double*>(smem_raw);   // [ROWS][C]
  double* ex = ring + ROWS * C;                          // owner: [NT][4] c0 c1 w0 w1 per head row
  double* rx = ex + 4 * NT;                              // holder: [NT][4] x~_c, x~_{c+1}
  double* s_al = rx + 4 * NT;                            // [stages][Q][4]
  double* s_ga = s_al + kPMaxStages * kPMaxQ * 4;
  double* s_fold = s_ga + kPMaxStages * kPMaxQ * 4;      // [Q][4]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(s_fold + kPMaxQ * 4);  // ring, ex, rx
  uint64_t* mbar_ex = mbar + 1;
  uint64_t* mbar_rx = mbar + 2;

  const int tid = threadIdx.x;
  const int Q = A.Q, G = A.G, stages = A.stages;
  const int j = tid % C, cl = tid / C;
  const uint32_t g = (G > 1) ? dev::cluster_ctarank() : 0u;
  const int c = (int)g * CPC + cl;
  const int cpo = C / G;
  const uint32_t owner = (uint32_t)(j / cpo);
  const int slot = (j % cpo) * Q + c;
  const int oj = tid / Q, oc = tid - (tid / Q) * Q;
  const int ocol = (int)g * cpo + oj;
  const int prev_row = oj * Q + ((oc - 1) & (Q - 1));
  const int ocm = (oc - 1) & (Q - 1);

  for (int i = tid; i < stages * Q * 4; i += NT) {
    s_al[i] = A.tab[i];
    s_ga[i] = A.tab[stages * Q * 4 + i];
  }
  for (int i = tid; i < Q * 4; i += NT) s_fold[i] = A.tab[2 * stages * Q * 4 + i];
  if (tid == 0) {
    dev::mbar_init(dev::smem_u32(mbar), 1);
    dev::mbar_init(dev::smem_u32(mbar_ex), 1);
    dev::mbar_init(dev::smem_u32(mbar_rx), 1);
    dev::fence_mbar_init();
  }
  __syncthreads();
  if (G > 1) dev::cluster_sync();

  const uint32_t ncl = (G > 1) ? dev::ncluster_x() : gridDim.x;
  const int64_t first = (G > 1) ? (int64_t)dev::cluster_id_x() : (int64_t)blockIdx.x;
  const uint64_t pol = dev::policy_evict_first();
  auto rmap = [&](const void* p, uint32_t rank) {
    const uint32_t a = dev::smem_u32(p);
    return G > 1 ? dev::mapa(a, rank) : a;
  };
  auto issue = [&](int64_t t) {
    if (t >= A.num_tiles) return;
    const int o = (int)(t / A.tiles_per_outer);
    const int col0 = (int)(t - (int64_t)o * A.tiles_per_outer) * C;
    const uint32_t bar = dev::smem_u32(mbar);
    dev::fence_proxy_async();
    dev::mbar_expect_tx(bar, (uint32_t)(ROWS * C * 8));
    dev::tma_load_3d(dev::smem_u32(ring), &tmap, col0, (int)g * ROWS, o, bar, pol);
  };
  if (tid == 0) issue(first);

  // measurement only (CTRI_TILE_TRACE): one CTA stamps the phases of its first 64 tiles
  unsigned long long* tr = (A.trace && (int)blockIdx.x == A.trace_cta) ? A.trace : nullptr;
  auto stamp = [&](int it_, int k) {
    if (tr && tid == 0 && it_ < 64) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      tr[it_ * 16 + k] = tt;
    }
  };
  int it = 0;
  for (int64_t t = first; t < A.num_tiles; t += ncl, ++it) {
    stamp(it, 0);
    const int64_t o = t / A.tiles_per_outer;
    const int64_t col = (t - o * A.tiles_per_outer) * C + j;
    if (tid == 0) {
      dev::mbar_expect_tx(dev::smem_u32(mbar_ex), (uint32_t)NT * 32u);
      dev::mbar_expect_tx(dev::smem_u32(mbar_rx), (uint32_t)NT * 32u);
    }
    dev::mbar_wait(dev::smem_u32(mbar), (uint32_t)it & 1u);
    double v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = ring[(cl * K + k) * C + j];
    stamp(it, 1);
    __syncthreads();  // the ring slot is free
    if (tid == 0) issue(t + ncl);
    const bool valid = col < A.lay.inner;

    // ---- register leaf: the pentadiagonal interior of the chunk (Eq. yi with r = 2) ----
    const double bt0 = v[0], bt1 = v[1];
    {
      double z1 = 0.0, z2 = 0.0;
#pragma unroll
      for (int k = 0; k < kPN; ++k) {
        const double z = v[k + 2] - T.lam1[k] * z1 - T.lam2[k] * z2;
        v[k + 2] = z;
        z2 = z1;
        z1 = z;
      }
      double y1 = 0.0, y2 = 0.0;
#pragma unroll
      for (int k = kPN - 1; k >= 0; --k) {
        const double y = (v[k + 2] - T.nu1[k] * y1 - T.f * y2) * T.imu[k];
        v[k + 2] = y;
        y2 = y1;
        y1 = y;
      }
    }
    stamp(it, 2);
    // chunk planes: c = b~ - U~ y, w = L~ y -> the owner of this column's head system
    {
      const uint32_t bar = rmap(mbar_ex, owner);
      const uint32_t dst = rmap(ex + 4 * slot, owner);
      dev::st_async_f64(dst, bt0 - T.f * v[2], bar);
      dev::st_async_f64(dst + 8, bt1 - (T.u * v[2] + T.f * v[3]), bar);
      dev::st_async_f64(dst + 16, T.e * v[K - 2] + T.l * v[K - 1], bar);
      dev::st_async_f64(dst + 24, T.e * v[K - 1], bar);
    }
    // ---- owner: b^_c = c_c - w_{c-1} (Eq. bi_hat), 2x2-block PCR over the Q heads ----
    {
      dev::mbar_wait(dev::smem_u32(mbar_ex), (uint32_t)it & 1u);
      stamp(it, 3);
      double h0 = ex[4 * tid], h1 = ex[4 * tid + 1];
      if (A.mode == 1 && oc == 0) {  // the partition's interface: decoupled dummy row
        h0 = 0.0;
        h1 = 0.0;
      } else if (!(A.mode == 2 && oc == 0)) {  // acyclic: no chunk above the first
        h0 -= ex[4 * prev_row + 2];
        h1 -= ex[4 * prev_row + 3];
      }
      if (Q <= 32) {  // the Q heads of a column are Q lanes of one warp: register shuffles
        for (int k = 0; k < stages; ++k) {
          const int sh = 1 << k;
          const int lm = (oc - sh) & (Q - 1), lp = (oc + sh) & (Q - 1);
          const double m0 = __shfl_sync(0xffffffffu, h0, lm, Q), m1 = __shfl_sync(0xffffffffu, h1, lm, Q);
          const double p0 = __shfl_sync(0xffffffffu, h0, lp, Q), p1 = __shfl_sync(0xffffffffu, h1, lp, Q);
          const double* a = s_al + (k * Q + oc) * 4;
          const double* gm = s_ga + (k * Q + oc) * 4;
          h0 = h0 - (a[0] * m0 + a[1] * m1) - (gm[0] * p0 + gm[1] * p1);
          h1 = h1 - (a[2] * m0 + a[3] * m1) - (gm[2] * p0 + gm[3] * p1);
        }
      } else {  // Q = 64: a column's heads span two warps; ping-pong through shared memory (the
                // exchange buffer, free once every owner has read its rows)
        __syncthreads();
        double* cur = ex;
        double* nxt = ex + 2 * NT;
        for (int k = 0; k < stages; ++k) {
          cur[2 * tid] = h0;
          cur[2 * tid + 1] = h1;
          __syncthreads();
          const int sh = 1 << k;
          const int rm = oj * Q + ((oc - sh) & (Q - 1)), rp = oj * Q + ((oc + sh) & (Q - 1));
          const double m0 = cur[2 * rm], m1 = cur[2 * rm + 1], p0 = cur[2 * rp], p1 = cur[2 * rp + 1];
          const double* a = s_al + (k * Q + oc) * 4;
          const double* gm = s_ga + (k * Q + oc) * 4;
          h0 = h0 - (a[0] * m0 + a[1] * m1) - (gm[0] * p0 + gm[1] * p1);
          h1 = h1 - (a[2] * m0 + a[3] * m1) - (gm[2] * p0 + gm[3] * p1);
          double* tmp = cur;
          cur = nxt;
          nxt = tmp;
        }
        __syncthreads();  // every read done before x~ leaves (the next tile's planes land here)
      }
      stamp(it, 4);
      const double* fo = s_fold + oc * 4;
      const double x0 = fo[0] * h0 + fo[1] * h1, x1 = fo[2] * h0 + fo[3] * h1;
      // x~_oc -> x~_c of chunk oc's holder and x~_{c+1} of chunk oc-1's holder
      const int ta = (oc % CPC) * C + ocol, tb = (ocm % CPC) * C + ocol;
      const uint32_t ra = rmap(rx + 4 * ta, (uint32_t)(oc / CPC));
      const uint32_t rb = rmap(rx + 4 * tb + 2, (uint32_t)(ocm / CPC));
      const uint32_t ba = rmap(mbar_rx, (uint32_t)(oc / CPC)), bb = rmap(mbar_rx, (uint32_t)(ocm / CPC));
      dev::st_async_f64(ra, x0, ba);
      dev::st_async_f64(ra + 8, x1, ba);
      dev::st_async_f64(rb, x0, bb);
      dev::st_async_f64(rb + 8, x1, bb);
    }
    dev::mbar_wait(dev::smem_u32(mbar_rx), (uint32_t)it & 1u);
    stamp(it, 5);
    const double xa0 = rx[4 * tid], xa1 = rx[4 * tid + 1];
    const bool last = (A.mode != 0 && c == Q - 1);  // x~_{c+1} lies outside D_i / acyclic end
    const double xb0 = last ? 0.0 : rx[4 * tid + 2], xb1 = last ? 0.0 : rx[4 * tid + 3];
    // ---- chunk back-substitution (Eq. xi_app, 2x2 blocks) ----
#pragma unroll
    for (int k = 0; k < kPN; ++k)
      v[k + 2] = v[k + 2] - (T.S0[k] * xa0 + T.S1[k] * xa1) - (T.R0[k] * xb0 + T.R1[k] * xb1);
    v[0] = (A.mode == 1 && c == 0) ? bt0 : xa0;  // mode 1: the interface rows keep b~ (scratch)
    v[1] = (A.mode == 1 && c == 0) ? bt1 : xa1;
    if (valid) {
      double* xp = A.x + (o * A.lay.n + (int64_t)c * K) * A.lay.inner + col;
#pragma unroll
      for (int k = 0; k < K; ++k) dev::st_global_cs(xp + (int64_t)k * A.lay.inner, v[k]);
      if (A.mode == 1) {  // the partition's planes c0 | c1 | w0 | w1 for the reduced system
        const int64_t pj = o * A.lay.inner + col;
        if (c == 0) {
          A.planes4[pj] = bt0 - T.f * v[2];
          A.planes4[A.pm + pj] = bt1 - (T.u * v[2] + T.f * v[3]);
        }
        if (c == Q - 1) {
          A.planes4[2 * A.pm + pj] = T.e * v[K - 2] + T.l * v[K - 1];
          A.planes4[3 * A.pm + pj] = T.e * v[K - 1];
        }
      }
    }
    stamp(it, 6);
  }
  if (G > 1) dev::cluster_sync();  // no CTA exits while peers may still address its smem
}

// ------------------------------------------------------------------------------------------
// host: configuration (chunk-level tables, head-system block PCR, occupancy) and launch
// ------------------------------------------------------------------------------------------
bool ptile_configure(Plan& P, std::string* why) {
  PTileConfig& pc = P.ptc;
  pc = PTileConfig();
  const Layout& L = P.tlay;
  if (L.inner < kPC || (L.inner % 2) != 0) { *why = "on-chip penta: strided axis with >= 32 columns"; return false; }
  if (L.n % (kPCPC * kPK) != 0) { *why = "on-chip penta: n not a multiple of 256"; return false; }
  const int G = (int)(L.n / (kPCPC * kPK));
  if (G < 1 || G > 8) { *why = "on-chip penta: n / 256 not in 1..8"; return false; }
  if (L.outer > ((int64_t)1 << 30) || L.inner > ((int64_t)1 << 31)) { *why = "dims too large"; return false; }
  const int Q = kPCPC * G;
  Penta cp;
  FactorError fe;
  if (!penta_factor(kPN, P.bands5, &cp, &fe)) { *why = "chunk penta factor: " + fe.detail; return false; }
  // head system of the Q chunks of a column: mode 0 cyclic uniform, mode 2 acyclic (first row
  // without a chunk above), mode 1 acyclic with the decoupled dummy row 0 (the partition's own
  // interface) and no coupling of row 1 to it
  const int mode = (P.p > 1 || P.vp > 1) ? 1 : (P.cyclic ? 0 : 2);
  std::vector<double> Lr(4 * (size_t)Q), Dr(4 * (size_t)Q), Ur(4 * (size_t)Q);
  for (int i = 0; i < Q; ++i)
    for (int e = 0; e < 4; ++e) {
      const bool lft = mode == 0 || i > (mode == 1 ? 1 : 0);
      const bool rgt = mode == 0 || i < Q - 1;
      Lr[4 * i + e] = lft ? cp.Lh[e] : 0.0;
      Dr[4 * i + e] = (mode == 2 && i == 0) ? cp.DhFirst[e] : cp.Dh[e];
      Ur[4 * i + e] = rgt ? cp.Uh[e] : 0.0;
    }
  if (mode == 1)
    for (int e = 0; e < 4; ++e) {
      Dr[e] = (e == 0 || e == 3) ? 1.0 : 0.0;
      Ur[e] = 0.0;
    }
  double mx = 0;
  for (int k = 0; k < 5; ++k) mx = std::max(mx, std::fabs(P.bands5[k]));
  PentaPcr t;
  if (!penta_block_pcr_rows(Q, mode == 0, Lr, Dr, Ur, 1e-13 * mx, &t, &fe)) {
    *why = "chunk head system: " + fe.detail;
    return false;
  }
  if (t.stages > kPMaxStages) { *why = "chunk head system: too many stages"; return false; }
  pc.tab.clear();
  pc.tab.insert(pc.tab.end(), t.alpha.begin(), t.alpha.end());
  pc.tab.insert(pc.tab.end(), t.gamma.begin(), t.gamma.end());
  pc.tab.insert(pc.tab.end(), t.fold.begin(), t.fold.end());
  pc.consts.clear();
  for (const std::vector<double>* vv : {&cp.lam1, &cp.lam2, &cp.nu1, &cp.inv_mu, &cp.S0, &cp.S1, &cp.R0, &cp.R1})
    pc.consts.insert(pc.consts.end(), vv->begin(), vv->end());
  pc.G = G;
  pc.Q = Q;
  pc.stages = t.stages;
  pc.mode = mode;
  pc.smem = (int)(sizeof(double) * ((size_t)kPCPC * kPK * kPC + 8 * kPNT + (2 * kPMaxStages + 1) * kPMaxQ * 4) + 3 * 8);
  if (cudaFuncSetAttribute(k_ptile, cudaFuncAttributeMaxDynamicSharedMemorySize, pc.smem) != cudaSuccess) {
    cudaGetLastError();
    *why = "cudaFuncSetAttribute(smem) failed";
    return false;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(kPNT, 1, 1);
  cfg.dynamicSmemBytes = pc.smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, k_ptile, &cfg) != cudaSuccess || nclusters < 1) {
    cudaGetLastError();
    *why = "on-chip penta: cluster occupancy query failed";
    return false;
  }
  const int64_t num_tiles = L.outer * ((L.inner + kPC - 1) / kPC);
  pc.grid = (int)(std::min<int64_t>(nclusters, num_tiles) * G);
  pc.ok = true;
  return true;
}

typedef CUresult (*EncodeTiledFnP)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t launch_ptile(const Plan& P, const double* b, double* x, cudaStream_t s) {
  const PTileConfig& pc = P.ptc;
  if (!pc.ok) return cudaErrorNotSupported;
  static EncodeTiledFnP enc = [] {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFnP) nullptr;
    return reinterpret_cast<EncodeTiledFnP>(fp);
  }();
  if (!enc) return cudaErrorNotSupported;
  const Layout& L = P.tlay;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  cuuint64_t gdim[3] = {(cuuint64_t)L.inner, (cuuint64_t)L.n, (cuuint64_t)L.outer};
  cuuint64_t gstride[2] = {(cuuint64_t)L.inner * 8, (cuuint64_t)(L.n * L.inner * 8)};
  cuuint32_t box[3] = {(cuuint32_t)kPC, (cuuint32_t)(kPCPC * kPK), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(b), gdim, gstride, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  PTileArgs A;
  A.x = x;
  A.lay = L;
  A.tiles_per_outer = (L.inner + kPC - 1) / kPC;
  A.num_tiles = L.outer * A.tiles_per_outer;
  A.Q = pc.Q;
  A.G = pc.G;
  A.stages = pc.stages;
  A.mode = pc.mode;
  A.tab = pc.d_tab;
  A.planes4 = P.d_planes4;
  A.pm = L.outer * L.inner;
  PTileConsts T;
  const double* cs = pc.consts.data();
  for (int k = 0; k < kPN; ++k) {
    T.lam1[k] = cs[k];
    T.lam2[k] = cs[kPN + k];
    T.nu1[k] = cs[2 * kPN + k];
    T.imu[k] = cs[3 * kPN + k];
    T.S0[k] = cs[4 * kPN + k];
    T.S1[k] = cs[5 * kPN + k];
    T.R0[k] = cs[6 * kPN + k];
    T.R1[k] = cs[7 * kPN + k];
  }
  T.e = P.bands5[0];
  T.l = P.bands5[1];
  T.u = P.bands5[3];
  T.f = P.bands5[4];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pc.grid, 1, 1);
  cfg.blockDim = dim3(kPNT, 1, 1);
  cfg.dynamicSmemBytes = pc.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pc.G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  A.trace = nullptr;
  A.trace_cta = 0;
  if (knob_tile_trace()) {  // measurement only
    static unsigned long long* d_tr = nullptr;
    if (!d_tr) cudaMalloc(&d_tr, 64 * 16 * sizeof(unsigned long long));
    cudaMemsetAsync(d_tr, 0, 64 * 16 * sizeof(unsigned long long), s);
    A.trace = d_tr;
    A.trace_cta = std::atoi(std::getenv("CTRI_TILE_TRACE"));
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_ptile, map, A, T);
  if (A.trace && e == cudaSuccess) {  // measurement only: the traced CTA's per-phase averages
    std::vector<unsigned long long> h(64 * 16);
    cudaMemcpyAsync(h.data(), A.trace, h.size() * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double acc[8] = {0};
    int cnt = 0;
    for (int i = 4; i < 60; ++i) {
      if (!h[i * 16 + 6] || !h[(i + 1) * 16]) break;
      for (int k = 1; k <= 6; ++k) acc[k] += (double)(h[i * 16 + k] - h[i * 16 + k - 1]);
      acc[7] += (double)(h[(i + 1) * 16] - h[i * 16 + 6]);
      ++cnt;
    }
    if (cnt)
      std::fprintf(stderr,
                   "[ptile trace] per tile (ns): ring_wait+lds %.0f leaf %.0f ex_wait %.0f pcr %.0f "
                   "rx_wait %.0f backsub+store %.0f loop %.0f total %.0f (%d tiles)\n",
                   acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt, acc[6] / cnt,
                   acc[7] / cnt, (acc[1] + acc[2] + acc[3] + acc[4] + acc[5] + acc[6] + acc[7]) / cnt, cnt);
  }
  return e;
}

}  // namespace ctri
