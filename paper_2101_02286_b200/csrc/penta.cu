// penta.cu -- the partition method for PENTADIAGONAL systems (r = 2).
//
// for a system of bandwidth w = 2r + 1 the interface block D~_i is r x r ("for a
// penta-diagonal system (w = 5), D~_i is 2x2"), L~_i / U~_i are short fat blocks and L_i / U_i
// tall skinny ones; Eqs. Si, Ri, Li_hat..Ui_hat, bi_hat and xi_app hold unchanged
// with 2x2 blocks, and "only the last r columns ... are needed for neighbor communication"
// (P:345).  Per partition of n rows (rows 0, 1 = x~_i, rows 2..n-1 = interior, N = n - 2):
//   (a1) k_penta_local: y_i = D_i^{-1} b_i by the plan-time LU factors of the pentadiagonal
//        interior (forward into x, backward in place), plus the planes c = b~_i - U~ y_i and
//        w = L~ y_i (2 values each); with one partition the 2x2 closure
//        (L^ + D^ + U^) x~ = c - w (cyclic) or D^ x~ = c (acyclic) is solved in place;
//   (a2)+(a3) p > 1: k_reduced_allgather_r2 (p2p.cu): one all-gather round of the 4 planes,
//        b^_r = c_r - w_{r-1}, x~_i and x~_{i+1} from plan-time rows of the 2p x 2p inverse;
//   (a4) k_penta_window: x = y - S x~_i - R x~_{i+1} on the window rows (reading R15, r = 2).
// HBM traffic of the column-serial local solve: b read once, the forward result written and
// read back once, y written once (32 B per point) -- DESIGN.md section 4.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"
#include "ptx.cuh"

namespace ctri {

struct PentaArgs {
  const double* b;
  double* x;
  int64_t outer, n, inner;
  const double* lu;   // [4][N]: lam1 | lam2 | nu1 | inv_mu
  double e, l, u, f;
  double* planes4;    // [4][m]
  int closure, cyclic;
  double cinv[4];     // p == 1: 2x2 closure inverse (row-major)
  int64_t k0c;        // LU factors are bitwise constant from interior row k0c on (plan-time)
  double c_lam1, c_lam2, c_nu1, c_imu;
};

constexpr int kPentaRows = 8;  // rows per batch (window kernel)
constexpr int kPB = 8;         // local solve: rows per register batch, next batch in flight

__global__ void __launch_bounds__(128, 4) k_penta_local(const PentaArgs A) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t m = A.outer * A.inner;
  if (j >= m) return;
  const int64_t o = j / A.inner, c = j - o * A.inner, st = A.inner;
  const int64_t N = A.n - 2;
  const double* bc = A.b + o * A.n * st + c + 2 * st;  // interior row 0
  double* xc = A.x + o * A.n * st + c;
  double* xi = xc + 2 * st;
  const double* lam1 = A.lu;
  const double* lam2 = A.lu + N;
  const double* nu1 = A.lu + 2 * N;
  const double* imu = A.lu + 3 * N;
  const double bt0 = A.b[o * A.n * st + c];
  const double bt1 = A.b[(o * A.n + 1) * st + c];
  const int64_t nb = (N + kPB - 1) / kPB;
  // forward: z_k = b_k - lam1[k] z_{k-1} - lam2[k] z_{k-2}   (interior row k = slab row k + 2);
  // software pipelined: batch i+1 is loaded before batch i is eliminated
  double cur[kPB], nxt[kPB];
#pragma unroll
  for (int t = 0; t < kPB; ++t) cur[t] = t < N ? bc[t * st] : 0.0;
  double z1 = 0.0, z2 = 0.0;
  for (int64_t bi = 0; bi < nb; ++bi) {
    const int64_t k0 = bi * kPB;
    if (bi + 1 < nb) {
#pragma unroll
      for (int t = 0; t < kPB; ++t)
        if (k0 + kPB + t < N) nxt[t] = bc[(k0 + kPB + t) * st];
    }
    if (k0 >= A.k0c && k0 + kPB <= N) {  // converged factors: scalars, no table loads
#pragma unroll
      for (int t = 0; t < kPB; ++t) {
        const double z = cur[t] - A.c_lam1 * z1 - A.c_lam2 * z2;
        xi[(k0 + t) * st] = z;
        z2 = z1;
        z1 = z;
      }
    } else {
#pragma unroll
      for (int t = 0; t < kPB; ++t) {
        const int64_t k = k0 + t;
        if (k < N) {
          const double z = cur[t] - __ldg(lam1 + k) * z1 - __ldg(lam2 + k) * z2;
          xi[k * st] = z;
          z2 = z1;
          z1 = z;
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kPB; ++t) cur[t] = nxt[t];
  }
  // backward: y_k = (z_k - nu1[k] y_{k+1} - f y_{k+2}) / mu[k], same pipelining
  double y1 = 0.0, y2 = 0.0, ylast = 0.0, ylast2 = 0.0;
  {
    const int64_t k0 = (nb - 1) * kPB;
#pragma unroll
    for (int t = 0; t < kPB; ++t) cur[t] = k0 + t < N ? xi[(k0 + t) * st] : 0.0;
  }
  for (int64_t bi = nb - 1; bi >= 0; --bi) {
    const int64_t k0 = bi * kPB;
    if (bi > 0) {
#pragma unroll
      for (int t = 0; t < kPB; ++t) nxt[t] = xi[(k0 - kPB + t) * st];
    }
    if (k0 >= A.k0c && k0 + kPB < N - 1) {  // converged factors, not the last two rows
#pragma unroll
      for (int t = kPB - 1; t >= 0; --t) {
        const double y = (cur[t] - A.c_nu1 * y1 - A.f * y2) * A.c_imu;
        xi[(k0 + t) * st] = y;
        y2 = y1;
        y1 = y;
      }
    } else {
#pragma unroll
      for (int t = kPB - 1; t >= 0; --t) {
        const int64_t k = k0 + t;
        if (k < N) {
          const double y = (cur[t] - __ldg(nu1 + k) * y1 - A.f * y2) * __ldg(imu + k);
          xi[k * st] = y;
          if (k == N - 1) ylast = y;
          if (k == N - 2) ylast2 = y;
          y2 = y1;
          y1 = y;
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kPB; ++t) cur[t] = nxt[t];
  }
  // y1 = y[0], y2 = y[1];  planes: c = b~ - U~ y_i[0..1], w = L~ y_i[N-2..N-1]
  const double c0 = bt0 - A.f * y1;
  const double c1 = bt1 - (A.u * y1 + A.f * y2);
  const double w0 = A.e * ylast2 + A.l * ylast;
  const double w1 = A.e * ylast;
  if (A.closure) {  // one partition: x~ = (closure)^{-1} b^, b^ = c - w (cyclic) or c (acyclic)
    const double h0 = c0 - (A.cyclic ? w0 : 0.0), h1 = c1 - (A.cyclic ? w1 : 0.0);
    xc[0] = A.cinv[0] * h0 + A.cinv[1] * h1;
    xc[st] = A.cinv[2] * h0 + A.cinv[3] * h1;
  } else {
    A.planes4[j] = c0;
    A.planes4[m + j] = c1;
    A.planes4[2 * m + j] = w0;
    A.planes4[3 * m + j] = w1;
  }
}

// Contiguous solve axis (inner == 1): a column's rows are contiguous, so the column-serial
// thread-per-column walk would touch 32 columns n*8 bytes apart per warp access.  Blocks of
// 32 rows x 128 columns are moved through shared memory instead: lane l of a warp loads row l
// of 32 columns in turn (256-byte coalesced accesses), each thread then runs the recurrence on
// its own column out of shared memory, and the block is written back the same way.
constexpr int kPcRows = 32, kPcCols = 128, kPcPad = kPcRows + 1;

__global__ void __launch_bounds__(kPcCols) k_penta_local_contig(const PentaArgs A) {
  __shared__ double tile[kPcCols * kPcPad];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t col0 = (int64_t)blockIdx.x * kPcCols;
  const int64_t mcols = A.outer;  // contiguous axis: one column per outer index
  const int64_t n = A.n, N = n - 2;
  const int64_t j = col0 + tid;
  const bool valid = j < mcols;
  const double* lam1 = A.lu;
  const double* lam2 = A.lu + N;
  const double* nu1 = A.lu + 2 * N;
  const double* imu = A.lu + 3 * N;
  double* mycol = tile + tid * kPcPad;
  // move interior rows [k0, k0 + 32) of the CTA's columns between HBM and shared memory
  // the next block is fetched into registers (32 loads in flight per thread) while the current
  // one is eliminated out of shared memory
  double reg[32];
  auto fetch_block = [&](const double* src, int64_t k0) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int64_t cj = col0 + warp * 32 + i;
      const int64_t k = k0 + lane;
      reg[i] = (cj < mcols && k < N) ? src[cj * n + 2 + k] : 0.0;
    }
  };
  auto put_block = [&]() {
#pragma unroll
    for (int i = 0; i < 32; ++i) tile[(warp * 32 + i) * kPcPad + lane] = reg[i];
  };
  auto store_block = [&](int64_t k0) {
    for (int i = 0; i < 32; ++i) {
      const int cl = warp * 32 + i;
      const int64_t cj = col0 + cl;
      const int64_t k = k0 + lane;
      if (cj < mcols && k < N) A.x[cj * n + 2 + k] = tile[cl * kPcPad + lane];
    }
  };
  double bt0 = 0.0, bt1 = 0.0;
  if (valid) {
    bt0 = A.b[j * n];
    bt1 = A.b[j * n + 1];
  }
  double z1 = 0.0, z2 = 0.0;
  fetch_block(A.b, 0);
  for (int64_t k0 = 0; k0 < N; k0 += kPcRows) {
    put_block();
    __syncthreads();
    if (k0 + kPcRows < N) fetch_block(A.b, k0 + kPcRows);
    if (valid) {
      if (k0 >= A.k0c && k0 + kPcRows <= N) {  // converged factors
#pragma unroll
        for (int t = 0; t < kPcRows; ++t) {
          const double z = mycol[t] - A.c_lam1 * z1 - A.c_lam2 * z2;
          mycol[t] = z;
          z2 = z1;
          z1 = z;
        }
      } else {
        for (int t = 0; t < kPcRows && k0 + t < N; ++t) {
          const int64_t k = k0 + t;
          const double z = mycol[t] - __ldg(lam1 + k) * z1 - __ldg(lam2 + k) * z2;
          mycol[t] = z;
          z2 = z1;
          z1 = z;
        }
      }
    }
    __syncthreads();
    store_block(k0);
    __syncthreads();
  }
  double y1 = 0.0, y2 = 0.0, ylast = 0.0, ylast2 = 0.0;
  const int64_t nb = (N + kPcRows - 1) / kPcRows;
  fetch_block(A.x, (nb - 1) * kPcRows);
  for (int64_t bi = nb - 1; bi >= 0; --bi) {
    const int64_t k0 = bi * kPcRows;
    put_block();
    __syncthreads();
    if (bi > 0) fetch_block(A.x, k0 - kPcRows);
    if (valid) {
      if (k0 >= A.k0c && k0 + kPcRows < N - 1) {  // converged factors, not the last two rows
#pragma unroll
        for (int t = kPcRows - 1; t >= 0; --t) {
          const double y = (mycol[t] - A.c_nu1 * y1 - A.f * y2) * A.c_imu;
          mycol[t] = y;
          y2 = y1;
          y1 = y;
        }
      } else {
        for (int t = kPcRows - 1; t >= 0; --t) {
          const int64_t k = k0 + t;
          if (k >= N) continue;
          const double y = (mycol[t] - __ldg(nu1 + k) * y1 - A.f * y2) * __ldg(imu + k);
          mycol[t] = y;
          if (k == N - 1) ylast = y;
          if (k == N - 2) ylast2 = y;
          y2 = y1;
          y1 = y;
        }
      }
    }
    __syncthreads();
    store_block(k0);
    __syncthreads();
  }
  if (!valid) return;
  const double c0 = bt0 - A.f * y1;
  const double c1 = bt1 - (A.u * y1 + A.f * y2);
  const double w0 = A.e * ylast2 + A.l * ylast;
  const double w1 = A.e * ylast;
  if (A.closure) {
    const double h0 = c0 - (A.cyclic ? w0 : 0.0), h1 = c1 - (A.cyclic ? w1 : 0.0);
    A.x[j * n] = A.cinv[0] * h0 + A.cinv[1] * h1;
    A.x[j * n + 1] = A.cinv[2] * h0 + A.cinv[3] * h1;
  } else {
    A.planes4[j] = c0;
    A.planes4[mcols + j] = c1;
    A.planes4[2 * mcols + j] = w0;
    A.planes4[3 * mcols + j] = w1;
  }
}

struct PentaWinArgs {
  double* x;
  const double* SR;    // [4][N]: S0 | S1 | R0 | R1
  const double* next;  // [2][m] x~_{i+1} (p > 1), else nullptr
  int64_t outer, n, inner, N, W, rows;  // n: rows of one partition (a slab, or 1/vp of it)
  int full, wrap;
  int vp;              // partitions per slab (nparts == 1); the grid's z index is the partition
};

__device__ __forceinline__ int64_t penta_row(const PentaWinArgs& A, int64_t ry) {
  return A.full ? ry : (ry < A.W ? ry : A.N - 2 * A.W + ry);  // interior row index k
}

// x_k = y_k - S0[k] x~_i[0] - S1[k] x~_i[1] - R0[k] x~_{i+1}[0] - R1[k] x~_{i+1}[1]  (Eq. xi_app)
__device__ __forceinline__ double penta_fix(const PentaWinArgs& A, int64_t k, double y, double a0,
                                            double a1, double n0, double n1) {
  const double* S0 = A.SR;
  const double* S1 = A.SR + A.N;
  const double* R0 = A.SR + 2 * A.N;
  const double* R1 = A.SR + 3 * A.N;
  return y - (__ldg(S0 + k) * a0 + __ldg(S1 + k) * a1) - (__ldg(R0 + k) * n0 + __ldg(R1 + k) * n1);
}

__global__ void __launch_bounds__(256) k_penta_window(const PentaWinArgs A) {
  const int64_t j = blockIdx.x * 256ll + threadIdx.x;
  const int64_t m = A.outer * A.inner;
  if (j >= m) return;
  const int64_t o = j / A.inner, c = j - o * A.inner, st = A.inner;
  const int s = blockIdx.z;  // partition of the slab
  double* xc = A.x + (o * A.vp + s) * A.n * st + c;
  const double a0 = xc[0], a1 = xc[st];
  double n0 = 0.0, n1 = 0.0;
  if (s + 1 < A.vp) {  // x~ of the next partition on this GPU
    n0 = xc[A.n * st];
    n1 = xc[(A.n + 1) * st];
  } else if (A.next) {
    n0 = A.next[j];
    n1 = A.next[m + j];
  } else if (A.wrap) {  // the first partition of the slab (itself when vp == 1)
    const double* x0 = A.x + o * A.vp * A.n * st + c;
    n0 = x0[0];
    n1 = x0[st];
  }
  const int64_t r0 = (int64_t)blockIdx.y * kPentaRows;
  double v[kPentaRows];
#pragma unroll
  for (int t = 0; t < kPentaRows; ++t)
    if (r0 + t < A.rows) v[t] = xc[(penta_row(A, r0 + t) + 2) * st];
#pragma unroll
  for (int t = 0; t < kPentaRows; ++t)
    if (r0 + t < A.rows) {
      const int64_t k = penta_row(A, r0 + t);
      xc[(k + 2) * st] = penta_fix(A, k, v[t], a0, a1, n0, n1);
    }
}

// strided axis with an even row length: a thread owns a PAIR of adjacent columns (16-byte
// loads and stores) and kPentaRows consecutive window rows, all loads in flight before the
// first store (as k_window_pairs)
__global__ void __launch_bounds__(256) k_penta_window_pairs(const PentaWinArgs A) {
  const int64_t j = 2 * (blockIdx.x * 256ll + threadIdx.x);  // first column of the pair
  const int64_t m = A.outer * A.inner;
  if (j >= m) return;
  const int64_t o = j / A.inner, c = j - o * A.inner, st = A.inner;
  const int s = blockIdx.z;  // partition of the slab
  double* xc = A.x + (o * A.vp + s) * A.n * st + c;
  const double2 a0 = *reinterpret_cast<const double2*>(xc);
  const double2 a1 = *reinterpret_cast<const double2*>(xc + st);
  double2 n0 = make_double2(0.0, 0.0), n1 = make_double2(0.0, 0.0);
  if (s + 1 < A.vp) {  // x~ of the next partition on this GPU
    n0 = *reinterpret_cast<const double2*>(xc + A.n * st);
    n1 = *reinterpret_cast<const double2*>(xc + (A.n + 1) * st);
  } else if (A.next) {
    n0 = *reinterpret_cast<const double2*>(A.next + j);
    n1 = *reinterpret_cast<const double2*>(A.next + m + j);
  } else if (A.wrap) {  // the first partition of the slab (itself when vp == 1)
    const double* x0 = A.x + o * A.vp * A.n * st + c;
    n0 = *reinterpret_cast<const double2*>(x0);
    n1 = *reinterpret_cast<const double2*>(x0 + st);
  }
  const int64_t r0 = (int64_t)blockIdx.y * kPentaRows;
  double2 v[kPentaRows];
  double* pr[kPentaRows];
#pragma unroll
  for (int t = 0; t < kPentaRows; ++t) {
    pr[t] = xc + (penta_row(A, r0 + t) + 2) * st;
    if (r0 + t < A.rows) v[t] = *reinterpret_cast<const double2*>(pr[t]);
  }
#pragma unroll
  for (int t = 0; t < kPentaRows; ++t)
    if (r0 + t < A.rows) {
      const int64_t k = penta_row(A, r0 + t);
      const double s0 = __ldg(A.SR + k), s1 = __ldg(A.SR + A.N + k);
      const double q0 = __ldg(A.SR + 2 * A.N + k), q1 = __ldg(A.SR + 3 * A.N + k);
      dev::st_global_cs_v2(pr[t], v[t].x - (s0 * a0.x + s1 * a1.x) - (q0 * n0.x + q1 * n1.x),
                           v[t].y - (s0 * a0.y + s1 * a1.y) - (q0 * n0.y + q1 * n1.y));
    }
}

// contiguous solve axis: one warp per column, lanes along the rows
__global__ void __launch_bounds__(256) k_penta_window_contig(const PentaWinArgs A) {
  const int64_t w = blockIdx.x * 8ll + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= A.outer) return;
  double* xc = A.x + w * A.n;
  const double a0 = xc[0], a1 = xc[1];
  double n0 = 0.0, n1 = 0.0;
  if (A.next) {
    n0 = A.next[w];
    n1 = A.next[A.outer + w];
  } else if (A.wrap) {
    n0 = a0;
    n1 = a1;
  }
  for (int64_t ry = lane; ry < A.rows; ry += 32) {
    const int64_t k = penta_row(A, ry);
    xc[k + 2] = penta_fix(A, k, xc[k + 2], a0, a1, n0, n1);
  }
}

// ------------------------------------------------------------------------------------------
// plan set-up and solve
// ------------------------------------------------------------------------------------------
static ctri_status upload_vec(double** d, const std::vector<double>& h, cudaStream_t s) {
  if (cudaMalloc(d, sizeof(double) * std::max<size_t>(1, h.size())) != cudaSuccess)
    return CTRI_ERR_OOM;
  if (cudaMemcpyAsync(*d, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice, s) != cudaSuccess)
    return CTRI_ERR_CUDA;
  return CTRI_OK;
}

ctri_status penta_plan_tables(Plan* P, cudaStream_t s, std::string* why) {
  // the partitions the local kernel solves: the slab, or its vp partitions (nparts == 1)
  const int64_t n = P->tlay.n, N = n - 2, m = P->lay.m();
  FactorError fe;
  if (!penta_factor(N, P->bands5, &P->pt, &fe)) {
    *why = fe.detail;
    return (ctri_status)fe.code;
  }
  const Penta& pt = P->pt;
  P->window = penta_window(pt);
  double mx = 0;
  for (int k = 0; k < 5; ++k) mx = std::max(mx, std::fabs(P->bands5[k]));
  const double guard = 1e-13 * mx;
  std::vector<double> inv;
  if (!penta_reduced_inverse(P->p, P->cyclic != 0, pt, guard, &inv, &fe)) {
    *why = fe.detail;
    return (ctri_status)fe.code;
  }
  P->ainv = inv;
  if (P->p == 1) std::memcpy(P->pcinv, inv.data(), sizeof(P->pcinv));
  P->pdense = false;
  if (P->p == 1 && P->vp > 1) {  // 2x2-block PCR over the vp partitions of this GPU (R20)
    std::vector<double> t;
    if (P->cyclic && (P->vp & (P->vp - 1)) != 0) {
      // cyclic with vp not a power of two: the plan-time inverse of the 2vp x 2vp block system
      if (!penta_reduced_inverse(P->vp, true, pt, guard, &t, &fe)) {
        *why = fe.detail;
        return (ctri_status)fe.code;
      }
      P->vppcr = PentaPcr();
      P->pdense = true;
    } else {
      if (!penta_block_pcr(P->vp, P->cyclic != 0, pt, guard, &P->vppcr, &fe)) {
        *why = fe.detail;
        return (ctri_status)fe.code;
      }
      t.insert(t.end(), P->vppcr.alpha.begin(), P->vppcr.alpha.end());
      t.insert(t.end(), P->vppcr.gamma.begin(), P->vppcr.gamma.end());
      t.insert(t.end(), P->vppcr.fold.begin(), P->vppcr.fold.end());
    }
    if (P->d_vppcr) cudaFree(P->d_vppcr);
    P->d_vppcr = nullptr;
    ctri_status st = upload_vec(&P->d_vppcr, t, s);
    if (st != CTRI_OK) return st;
  }
  std::vector<double> lu, sr;
  for (const std::vector<double>* v : {&pt.lam1, &pt.lam2, &pt.nu1, &pt.inv_mu}) lu.insert(lu.end(), v->begin(), v->end());
  for (const std::vector<double>* v : {&pt.S0, &pt.S1, &pt.R0, &pt.R1}) sr.insert(sr.end(), v->begin(), v->end());
  ctri_status st;
  for (double** d : {&P->d_plu, &P->d_pSR, &P->d_ainv, &P->d_planes4})  // (called again when the
    if (*d) {                                                            //  partition size changes)
      cudaFree(*d);
      *d = nullptr;
    }
  if ((st = upload_vec(&P->d_plu, lu, s)) != CTRI_OK) return st;
  if ((st = upload_vec(&P->d_pSR, sr, s)) != CTRI_OK) return st;
  if ((st = upload_vec(&P->d_ainv, inv, s)) != CTRI_OK) return st;
  if (P->p == 1 && P->vp > 1 &&
      cudaMalloc(&P->d_planes4, sizeof(double) * 4 * m * P->vp) != cudaSuccess)
    return CTRI_ERR_OOM;
  if (P->p > 1) {  // per virtual row: planes [4][m * vp], x~ of the next block row [vp][2][m]
    if (P->d_xnext2) cudaFree(P->d_xnext2);
    P->d_xnext2 = nullptr;
    if (cudaMalloc(&P->d_planes4, sizeof(double) * 4 * m * P->vp) != cudaSuccess) return CTRI_ERR_OOM;
    if (cudaMalloc(&P->d_xnext2, sizeof(double) * 2 * m * P->vp) != cudaSuccess) return CTRI_ERR_OOM;
    if (cudaMemsetAsync(P->d_xnext2, 0, sizeof(double) * 2 * m * P->vp, s) != cudaSuccess) return CTRI_ERR_CUDA;
  }
  return CTRI_OK;
}

cudaError_t launch_penta_local(const Plan& P, const double* b, double* x, cudaStream_t s) {
  PentaArgs A;
  A.b = b;
  A.x = x;
  A.outer = P.lay.outer;
  A.n = P.lay.n;
  A.inner = P.lay.inner;
  A.lu = P.d_plu;
  A.e = P.bands5[0];
  A.l = P.bands5[1];
  A.u = P.bands5[3];
  A.f = P.bands5[4];
  A.planes4 = P.d_planes4;
  A.closure = P.p == 1 ? 1 : 0;
  A.cyclic = P.cyclic;
  std::memcpy(A.cinv, P.pcinv, sizeof(A.cinv));
  const Penta& pt = P.pt;
  const int64_t N = pt.N;
  A.k0c = N;  // first row from which all four factors equal their last value bitwise
  while (A.k0c > 0 && pt.lam1[A.k0c - 1] == pt.lam1[N - 1] && pt.lam2[A.k0c - 1] == pt.lam2[N - 1] &&
         pt.nu1[A.k0c - 1] == pt.nu1[N - 1] && pt.inv_mu[A.k0c - 1] == pt.inv_mu[N - 1])
    --A.k0c;
  A.k0c = std::max<int64_t>(A.k0c, 2);  // rows 0, 1 have lam2 = 0 / lam1 = 0 by construction
  A.c_lam1 = pt.lam1[N - 1];
  A.c_lam2 = pt.lam2[N - 1];
  A.c_nu1 = pt.nu1[N - 1];
  A.c_imu = pt.inv_mu[N - 1];
  const int64_t m = P.lay.m();
  if (P.lay.inner == 1)
    k_penta_local_contig<<<(unsigned)((m + kPcCols - 1) / kPcCols), kPcCols, 0, s>>>(A);
  else
    k_penta_local<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_penta_window(const Plan& P, double* x, cudaStream_t s) {
  PentaWinArgs A;
  A.x = x;
  A.SR = P.d_pSR;
  A.next = P.p > 1 ? P.d_xnext2 + (int64_t)(P.vp - 1) * 2 * P.lay.m() : nullptr;  // the last row's
  A.outer = P.lay.outer;
  A.n = P.tlay.n;
  A.inner = P.lay.inner;
  A.N = P.tlay.n - 2;
  A.vp = P.vp;
  A.W = P.window;
  A.full = ((P.flags & CTRI_FLAG_FULL_BACKSUB) || 2 * P.window >= A.N) ? 1 : 0;
  A.rows = A.full ? A.N : 2 * A.W;
  A.wrap = (P.p == 1 && P.cyclic) ? 1 : 0;
  if (A.rows <= 0) return cudaSuccess;
  if (A.inner == 1) {
    k_penta_window_contig<<<(unsigned)((A.outer + 7) / 8), 256, 0, s>>>(A);
  } else {
    const int64_t m = P.lay.m();
    const bool pairs = (A.inner % 2) == 0;
    const int64_t cpb = pairs ? 512 : 256;  // columns per block
    dim3 grid((unsigned)((m + cpb - 1) / cpb), (unsigned)((A.rows + kPentaRows - 1) / kPentaRows),
              (unsigned)A.vp);
    if (pairs) k_penta_window_pairs<<<grid, 256, 0, s>>>(A);
    else k_penta_window<<<grid, 256, 0, s>>>(A);
  }
  return cudaGetLastError();
}

// (a2)+(a3) across the vp partitions of one GPU (nparts == 1, local_kernel 4): per batch column
// b^_v = c_v - w_{v-1} (Eq. bi_hat with 2x2 blocks; cyclic wrap or none), 2x2-block PCR
// over the vp rows with the plan's multipliers (R20; fold R3) and x~_v into rows 0, 1 of
// partition v; the window pass follows.
__global__ void __launch_bounds__(128) k_penta_reduced_local(double* __restrict__ x,
                                                             const double* __restrict__ planes4,
                                                             const double* __restrict__ tab,
                                                             int64_t outer, int64_t nv, int64_t inner,
                                                             int vp, int stages, int cyclic, int dense) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t m = outer * inner;
  if (j >= m) return;
  const int64_t o = j / inner, c = j - o * inner, pm = m * vp;
  double b0[8], b1[8];
  for (int v = 0; v < vp; ++v) {
    const int64_t pj = (o * vp + v) * inner + c;
    const int vl = v == 0 ? vp - 1 : v - 1;
    const int64_t pl = (o * vp + vl) * inner + c;
    const bool lft = cyclic || v > 0;
    b0[v] = planes4[pj] - (lft ? planes4[2 * pm + pl] : 0.0);
    b1[v] = planes4[pm + pj] - (lft ? planes4[3 * pm + pl] : 0.0);
  }
  if (dense) {  // cyclic, vp not a power of two: x~ = (A^)^-1 b^ with the plan-time inverse
                // (block row v, component r at index 2v + r)
    const int n2 = 2 * vp;
    for (int v = 0; v < vp; ++v) {
      double a0 = 0.0, a1 = 0.0;
      for (int w = 0; w < vp; ++w) {
        a0 += tab[(2 * v) * n2 + 2 * w] * b0[w] + tab[(2 * v) * n2 + 2 * w + 1] * b1[w];
        a1 += tab[(2 * v + 1) * n2 + 2 * w] * b0[w] + tab[(2 * v + 1) * n2 + 2 * w + 1] * b1[w];
      }
      double* xs = x + (o * vp + v) * nv * inner + c;
      xs[0] = a0;
      xs[inner] = a1;
    }
    return;
  }
  for (int k = 0; k < stages; ++k) {
    const int sh = 1 << k;
    double n0[8], n1[8];
    for (int v = 0; v < vp; ++v) {
      int im = v - sh, ip = v + sh;
      double m0 = 0.0, m1 = 0.0, p0 = 0.0, p1 = 0.0;
      if (cyclic) {
        im = ((im % vp) + vp) % vp;
        ip = ip % vp;
      }
      if (im >= 0) { m0 = b0[im]; m1 = b1[im]; }
      if (ip < vp) { p0 = b0[ip]; p1 = b1[ip]; }
      const double* a = tab + ((size_t)k * vp + v) * 4;
      const double* g = tab + ((size_t)(stages + k) * vp + v) * 4;
      n0[v] = b0[v] - (a[0] * m0 + a[1] * m1) - (g[0] * p0 + g[1] * p1);
      n1[v] = b1[v] - (a[2] * m0 + a[3] * m1) - (g[2] * p0 + g[3] * p1);
    }
    for (int v = 0; v < vp; ++v) {
      b0[v] = n0[v];
      b1[v] = n1[v];
    }
  }
  for (int v = 0; v < vp; ++v) {
    const double* f = tab + ((size_t)2 * stages * vp + v) * 4;
    double* xs = x + (o * vp + v) * nv * inner + c;
    xs[0] = f[0] * b0[v] + f[1] * b1[v];
    xs[inner] = f[2] * b0[v] + f[3] * b1[v];
  }
}

cudaError_t launch_penta_reduced_local(const Plan& P, double* x, cudaStream_t s) {
  const int64_t m = P.lay.m();
  k_penta_reduced_local<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(
      x, P.d_planes4, P.d_vppcr, P.lay.outer, P.tlay.n, P.lay.inner, P.vp, P.vppcr.stages, P.cyclic,
      P.pdense ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace ctri
