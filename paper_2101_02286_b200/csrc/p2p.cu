// p2p.cu -- fused, device-initiated reduced phase (a2)-(a4) for nparts > 1.
//
// One kernel per solve replaces the host-issued NCCL rounds.  For its batch columns every
// thread
//   (a2) stores y_D[n-1] into the right neighbour's mailbox and forms
//        b^_i = b~_i - l y_{i-1}[last] - u y_i[first]                    (Eq. bi_hat)
//   (a3) runs the log2 p cyclic PCR stages: stores b^ into the mailboxes of ranks i +- 2^k,
//        waits for theirs, b^ <- b^ - alpha b^_{i-s} - gamma b^_{i+s}
//        and x~ = b^ / (L+D+U) after the fold (R3)
//   (a4) stores x~_i into the left neighbour's mailbox, waits for x~_{i+1} and applies
//        x_i = y_i - S_i x~_i - R_i x~_{i+1} on the window rows          (Eq. xi_app)
//
// Messages are "LL" words: each fp64 travels as two 8-byte words {32-bit half, 32-bit epoch}
// written with one 16-byte store over NVLink into CUDA-IPC-mapped peer memory.  An 8-byte
// word is single-copy atomic, so a receiver that sees the current epoch in both words has
// the value: no fences, no flags, no CTA barriers -- each thread polls only its own columns
// in its own (local) mailbox.  Mailboxes are double-buffered by epoch parity, so a word for
// solve e+1 never overwrites one of solve e that may still be unread.  Every wait has a
// deadline (%globaltimer), after which the kernel records an error and returns.
//
// Loopback test mode (all ranks on one GPU) launches every rank's CTAs in ONE cooperative
// grid, so no two kernels wait on each other.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "internal.h"
#include "ptx.cuh"

namespace ctri {

namespace {
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kP2PThreads = 256;
constexpr int kMaxCpt = 4;  // columns per thread (compile-time indexed: registers only)

// LL send: value + epoch tag as two 8-byte words in one 16-byte store (peer memory).
__device__ __forceinline__ void ll_send(unsigned long long* dst, double v, uint32_t ep) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const unsigned long long w0 = ((unsigned long long)ep << 32) | (bits & 0xffffffffull);
  const unsigned long long w1 = ((unsigned long long)ep << 32) | (bits >> 32);
  asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(dst), "l"(w0), "l"(w1)
               : "memory");
}

// LL receive: spin on the local word pair until both halves carry `ep` (false on deadline).
__device__ __forceinline__ bool ll_recv(const unsigned long long* src, uint32_t ep,
                                        unsigned long long deadline, double* out) {
  unsigned long long w0, w1;
  int spins = 0;
  while (true) {
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(w0), "=l"(w1) : "l"(src)
                 : "memory");
    if ((uint32_t)(w0 >> 32) == ep && (uint32_t)(w1 >> 32) == ep) break;
    if (++spins == 64) {
      spins = 0;
      if (globaltimer() > deadline) return false;
    }
  }
  *out = __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
  return true;
}
// Batched LL receive of the words at src + r * stride for the ranks r in `mask` (r < kMaxAG):
// every sweep issues all pending loads before testing any, so the waits overlap.
__device__ __forceinline__ bool ll_recv_batch(const unsigned long long* src, int64_t stride,
                                              uint32_t mask, uint32_t ep, unsigned long long deadline,
                                              double (&v)[kMaxAG]) {
  int spins = 0;
  while (mask) {
    unsigned long long w0[kMaxAG], w1[kMaxAG];
#pragma unroll
    for (int k = 0; k < kMaxAG; ++k)
      if (mask & (1u << k))
        asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];"
                     : "=l"(w0[k]), "=l"(w1[k]) : "l"(src + k * stride) : "memory");
#pragma unroll
    for (int k = 0; k < kMaxAG; ++k)
      if ((mask & (1u << k)) && (uint32_t)(w0[k] >> 32) == ep && (uint32_t)(w1[k] >> 32) == ep) {
        v[k] = __longlong_as_double((long long)((w1[k] << 32) | (w0[k] & 0xffffffffull)));
        mask &= ~(1u << k);
      }
    if (mask && ++spins == 64) {
      spins = 0;
      if (globaltimer() > deadline) return false;
    }
  }
  return true;
}
}  // namespace

__global__ void __launch_bounds__(kP2PThreads, 2)
    k_reduced_p2p(const P2PArgs A) {
  if (A.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");  // launched early (PDL)
  const int r_local = blockIdx.x / A.nslices;
  const int slice = blockIdx.x - r_local * A.nslices;
  const P2PRank& R = A.rk[r_local];
  const int p = A.p, q = A.q, rank = R.rank;
  const int64_t m = A.m;
  const int64_t c0 = (int64_t)slice * A.slice_cols;
  const int64_t c1 = std::min<int64_t>(m, c0 + A.slice_cols);
  // epoch of this solve: every rank runs the same sequence of solves, so slice `slice` of every
  // rank reads the same value; only this CTA touches its slot (written back at the end)
  const uint32_t ep = R.epoch[slice] + 1u;
  const unsigned long long deadline = globaltimer() + A.deadline_ns;
  // mailbox copy (epoch parity): [y: 2m][stage k, slot 0/1: 2m each][x: 2m] 64-bit words
  const int64_t copy_off = (int64_t)(ep & 1u) * A.copy_words;
  const int64_t OFF_Y = 0, OFF_X = (int64_t)(1 + 2 * q) * 2 * m;
  auto OFF_S = [&](int k, int slot) -> int64_t { return (int64_t)(1 + 2 * k + slot) * 2 * m; };
  const bool cyc = A.cyclic != 0;
  const int right = cyc ? (rank + 1) % p : (rank + 1 < p ? rank + 1 : -1);
  const int left = cyc ? (rank + p - 1) % p : (rank > 0 ? rank - 1 : -1);
  unsigned long long* const mine = R.mbox + copy_off;

  unsigned long long* tr = A.trace ? A.trace + (size_t)blockIdx.x * kP2PTrace : nullptr;
  auto stamp = [&](int k) {
    if (tr && threadIdx.x == 0) tr[k] = globaltimer();
  };
  stamp(kTrStart);
  bool ok = true;
  const int64_t n = A.lay.n, inner = A.lay.inner;
  // the slice's columns in batches of kMaxCpt per thread (one batch unless the grid had to be
  // capped to a single wave of co-resident CTAs)
  for (int64_t b0 = c0; b0 < c1 && ok; b0 += (int64_t)kP2PThreads * kMaxCpt) {
  const int64_t b1 = std::min<int64_t>(c1, b0 + (int64_t)kP2PThreads * kMaxCpt);
  double bh[kMaxCpt];
  int64_t col[kMaxCpt];
  int nc = 0;
#pragma unroll
  for (int i = 0; i < kMaxCpt; ++i) {
    const int64_t j = b0 + threadIdx.x + (int64_t)i * kP2PThreads;
    col[i] = j;
    if (j < b1) nc = i + 1;
  }
  // ---- (a2) y_i[last] -> right neighbour; b^ ----
  // the batch's planes into registers first: the LL stores are asm volatile with a memory
  // clobber, so no load can move across them (a load per store would serialise HBM latencies)
  double ylv[kMaxCpt], btv[kMaxCpt], yfv[kMaxCpt];
#pragma unroll
  for (int i = 0; i < kMaxCpt; ++i) {
    ylv[i] = btv[i] = yfv[i] = 0.0;
    if (i < nc) {
      ylv[i] = R.yl[col[i]];
      btv[i] = R.bt[col[i]];
      yfv[i] = R.yf[col[i]];
    }
  }
  if (right >= 0 && rank != A.test_drop_rank) {  // (test knob: a rank that never sends)
    unsigned long long* dst = R.peer_mbox[right] + copy_off + OFF_Y;
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i)
      if (i < nc) ll_send(dst + 2 * col[i], ylv[i], ep);
  }
  stamp(kTrYSent);
  {  // batched receive: every pending column's word is loaded before any is tested
    double ylp[kMaxCpt];
    uint32_t pend = 0;
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i) {
      ylp[i] = 0.0;
      if (i < nc && left >= 0) pend |= 1u << i;
    }
    int spins = 0;
    while (pend && ok) {
      unsigned long long w0[kMaxCpt], w1[kMaxCpt];
#pragma unroll
      for (int i = 0; i < kMaxCpt; ++i)
        if (pend & (1u << i)) dev::ll_load(mine + OFF_Y + 2 * col[i], &w0[i], &w1[i]);
#pragma unroll
      for (int i = 0; i < kMaxCpt; ++i)
        if ((pend & (1u << i)) && dev::ll_ready(w0[i], w1[i], ep)) {
          ylp[i] = dev::ll_value(w0[i], w1[i]);
          pend &= ~(1u << i);
        }
      if (pend && ++spins == 64) {
        spins = 0;
        if (globaltimer() > deadline) ok = false;
      }
    }
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i) bh[i] = btv[i] - A.l * ylp[i] - A.u * yfv[i];
  }
  stamp(kTrYRecv);
  // ---- (a3) reduced-system schedule: PCR stages, or detach / PCR / fold /
  //      reattach for cyclic non-power-of-two p; the fold is the last PCR step ----
  for (int s = 0; s < q && ok; ++s) {
    const P2PStep& S = R.step[s];
    if (S.dst0 >= 0) {
      unsigned long long* dst = R.peer_mbox[S.dst0] + copy_off + OFF_S(s, S.dslot0);
#pragma unroll
      for (int i = 0; i < kMaxCpt; ++i)
        if (i < nc) ll_send(dst + 2 * col[i], bh[i], ep);
    }
    if (S.dst1 >= 0) {
      unsigned long long* dst = R.peer_mbox[S.dst1] + copy_off + OFF_S(s, S.dslot1);
#pragma unroll
      for (int i = 0; i < kMaxCpt; ++i)
        if (i < nc) ll_send(dst + 2 * col[i], bh[i], ep);
    }
    // batched receive: every pending (column, source) word is loaded in one sweep before any
    // is tested, so the two partners' (and the columns') poll latencies overlap
    double u[2][kMaxCpt];
    uint32_t pend = 0;
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i) {
      u[0][i] = u[1][i] = 0.0;
      if (i < nc) pend |= (S.src0 >= 0 ? 1u : 0u) << (2 * i) | (S.src1 >= 0 ? 2u : 0u) << (2 * i);
    }
    int spins = 0;
    while (pend && ok) {
      unsigned long long w0[2 * kMaxCpt], w1[2 * kMaxCpt];
#pragma unroll
      for (int k = 0; k < 2 * kMaxCpt; ++k)
        if (pend & (1u << k)) dev::ll_load(mine + OFF_S(s, k & 1) + 2 * col[k >> 1], &w0[k], &w1[k]);
#pragma unroll
      for (int k = 0; k < 2 * kMaxCpt; ++k)
        if ((pend & (1u << k)) && dev::ll_ready(w0[k], w1[k], ep)) {
          u[k & 1][k >> 1] = dev::ll_value(w0[k], w1[k]);
          pend &= ~(1u << k);
        }
      if (pend && ++spins == 64) {
        spins = 0;
        if (globaltimer() > deadline) ok = false;
      }
    }
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i)
      if (i < nc) bh[i] = S.w * bh[i] - S.c0 * u[0][i] - S.c1 * u[1][i];
    stamp(kTrStep0 + s);
  }
  // (per-step stamps inside the loop)
  // ---- (a4) x~_i -> left neighbour; back-substitution on the window ----
  if (ok && left >= 0) {
    unsigned long long* dst = R.peer_mbox[left] + copy_off + OFF_X;
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i)
      if (i < nc) ll_send(dst + 2 * col[i], bh[i], ep);
  }
  double xb[kMaxCpt];
  {  // batched receive of x~_{i+1}
    uint32_t pend = 0;
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i) {
      xb[i] = 0.0;
      if (i < nc && right >= 0) pend |= 1u << i;
    }
    int spins = 0;
    while (pend && ok) {
      unsigned long long w0[kMaxCpt], w1[kMaxCpt];
#pragma unroll
      for (int i = 0; i < kMaxCpt; ++i)
        if (pend & (1u << i)) dev::ll_load(mine + OFF_X + 2 * col[i], &w0[i], &w1[i]);
#pragma unroll
      for (int i = 0; i < kMaxCpt; ++i)
        if ((pend & (1u << i)) && dev::ll_ready(w0[i], w1[i], ep)) {
          xb[i] = dev::ll_value(w0[i], w1[i]);
          pend &= ~(1u << i);
        }
      if (pend && ++spins == 64) {
        spins = 0;
        if (globaltimer() > deadline) ok = false;
      }
    }
  }
  if (!ok) {
    *reinterpret_cast<volatile int*>(A.err) = 1;
    break;
  }
  stamp(kTrXRecv);
  // x~_i into row 0 of this slab and x~_{i+1} into the next-plane; the window pass (k_window)
  // follows as its own high-occupancy launch
#pragma unroll
  for (int i = 0; i < kMaxCpt; ++i) {
    if (i >= nc) continue;
    const int64_t j = col[i];
    const int64_t o = j / inner, c = j - o * inner;
    R.x[o * n * inner + c] = bh[i];
    R.xnext[j] = xb[i];
  }
  }  // column batches
  __syncthreads();  // every thread has read this solve's epoch
  if (threadIdx.x == 0) R.epoch[slice] = ep;
  if (tr) stamp(kTrEnd);
}

// All-gather variant of (a2)-(a3) (CTRI_FLAG_ALLGATHER): one exchange round
// instead of 2 + log2 p dependent ones; its own kernel so each variant keeps its registers.
__global__ void __launch_bounds__(kP2PThreads, 1)
    k_reduced_allgather(const P2PArgs A) {
  if (A.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");  // launched early (PDL)
  const int r_local = blockIdx.x / A.nslices;
  const int slice = blockIdx.x - r_local * A.nslices;
  const P2PRank& R = A.rk[r_local];
  const int p = A.p, rank = R.rank;
  const int64_t m = A.m;
  const int64_t c0 = (int64_t)slice * A.slice_cols;
  const int64_t c1 = std::min<int64_t>(m, c0 + A.slice_cols);
  const uint32_t ep = R.epoch[slice] + 1u;
  const unsigned long long deadline = globaltimer() + A.deadline_ns;
  const int64_t copy_off = (int64_t)(ep & 1u) * A.copy_words;
  const bool cyc = A.cyclic != 0;
  unsigned long long* const mine = R.mbox + copy_off;
  unsigned long long* tr = A.trace ? A.trace + (size_t)blockIdx.x * kP2PTrace : nullptr;
  auto stamp = [&](int k) {
    if (tr && threadIdx.x == 0) tr[k] = globaltimer();
  };
  stamp(kTrStart);
  bool ok = true;
  const int64_t n = A.lay.n, inner = A.lay.inner;
  // ---- (a2)+(a3) as ONE round: c_i = b~_i - u y_i[first] and y_i[last] go to
  //      every peer; every rank forms all b^_r = c_r - l y_{r-1}[last] (Eq. bi_hat) and
  //      evaluates x~_i, x~_{i+1} with two plan-time rows of A^{-1} (no x~ round) ----
#pragma unroll 1
  for (int64_t j = c0 + threadIdx.x; j < c1; j += kP2PThreads) {
    const double cv = R.bt[j] - A.u * R.yf[j], yl = R.yl[j];
    for (int r = 0; r < p; ++r) {
      if (r == rank) continue;
      unsigned long long* dst = R.peer_mbox[r] + copy_off;
      ll_send(dst + (int64_t)rank * 2 * m + 2 * j, cv, ep);
      ll_send(dst + (int64_t)(p + rank) * 2 * m + 2 * j, yl, ep);
    }
  }
  stamp(kTrYSent);
#pragma unroll 1
  for (int64_t j = c0 + threadIdx.x; j < c1 && ok; j += kP2PThreads) {  // 2 x 8 loads in flight
    double c[kMaxAG], y[kMaxAG];
    uint32_t mask = 0;
#pragma unroll
    for (int r = 0; r < kMaxAG; ++r) {
      c[r] = y[r] = 0.0;
      if (r < p && r != rank) mask |= 1u << r;
    }
    ok = ll_recv_batch(mine + 2 * j, 2 * m, mask, ep, deadline, c) &&
         ll_recv_batch(mine + (int64_t)p * 2 * m + 2 * j, 2 * m, mask, ep, deadline, y);
    if (!ok) continue;
#pragma unroll
    for (int r = 0; r < kMaxAG; ++r)
      if (r == rank) { c[r] = R.bt[j] - A.u * R.yf[j]; y[r] = R.yl[j]; }
    double ywrap = 0.0;  // y_{p-1}[last], the left neighbour of rank 0 (cyclic)
#pragma unroll
    for (int r = 0; r < kMaxAG; ++r)
      if (r == p - 1 && cyc) ywrap = y[r];
    double xt = 0.0, xn = 0.0;
#pragma unroll
    for (int r = 0; r < kMaxAG; ++r) {
      if (r >= p) continue;
      const double bh_r = c[r] - A.l * (r > 0 ? y[r > 0 ? r - 1 : 0] : ywrap);  // Eq. bi_hat
      xt += R.ag0[r] * bh_r;
      xn += R.ag1[r] * bh_r;
    }
    const int64_t o = j / inner, cc = j - o * inner;
    R.x[o * n * inner + cc] = xt;
    R.xnext[j] = xn;
  }
  if (!ok) *reinterpret_cast<volatile int*>(A.err) = 1;
  __syncthreads();
  if (threadIdx.x == 0) R.epoch[slice] = ep;
  stamp(kTrYRecv);
  stamp(kTrXRecv);
  stamp(kTrEnd);
}

// Pentadiagonal (r = 2) reduced phase, all-gather form (SURVEY 8(f) N3 + N4): per column every
// rank sends its 4 plane values c = b~_i - U~ y_i (2) and w = L~ y_i[last two] (2) to every peer,
// forms the 2x2-block right-hand sides b^_r = c_r - w_{r-1} (Eq. bi_hat with r = 2) and
// evaluates x~_i, x~_{i+1} (2 values each) with plan-time rows of the 2p x 2p inverse of A^.
__global__ void __launch_bounds__(kP2PThreads, 1)
    k_reduced_allgather_r2(const P2PArgs A) {
  const int r_local = blockIdx.x / A.nslices;
  const int slice = blockIdx.x - r_local * A.nslices;
  const P2PRank& R = A.rk[r_local];
  const int p = A.p, rank = R.rank;
  const int64_t m = A.m;
  const int64_t c0 = (int64_t)slice * A.slice_cols;
  const int64_t c1 = std::min<int64_t>(m, c0 + A.slice_cols);
  const uint32_t ep = R.epoch[slice] + 1u;
  const unsigned long long deadline = globaltimer() + A.deadline_ns;
  const int64_t copy_off = (int64_t)(ep & 1u) * A.copy_words;
  const bool cyc = A.cyclic != 0;
  unsigned long long* const mine = R.mbox + copy_off;
  const int64_t n = A.lay.n, inner = A.lay.inner;
  const int nx = rank + 1 < p ? rank + 1 : (cyc ? 0 : -1);  // owner of x~_{i+1}
  unsigned long long* tr = A.trace ? A.trace + (size_t)blockIdx.x * kP2PTrace : nullptr;
  auto stamp = [&](int k) {
    if (tr && threadIdx.x == 0) tr[k] = globaltimer();
  };
  stamp(kTrStart);
  bool ok = true;
#pragma unroll 1
  for (int64_t j = c0 + threadIdx.x; j < c1; j += kP2PThreads) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = R.planes4[q * m + j];
    for (int r = 0; r < p; ++r) {
      if (r == rank) continue;
      unsigned long long* dst = R.peer_mbox[r] + copy_off;
#pragma unroll
      for (int q = 0; q < 4; ++q) ll_send(dst + (int64_t)(q * p + rank) * 2 * m + 2 * j, v[q], ep);
    }
  }
#pragma unroll 1
  for (int64_t j = c0 + threadIdx.x; j < c1 && ok; j += kP2PThreads) {
    double pl[4][kMaxAG];
    uint32_t mask = 0;
#pragma unroll
    for (int r = 0; r < kMaxAG; ++r) {
      if (r < p && r != rank) mask |= 1u << r;
#pragma unroll
      for (int q = 0; q < 4; ++q) pl[q][r] = 0.0;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      ok = ok && ll_recv_batch(mine + (int64_t)q * p * 2 * m + 2 * j, 2 * m, mask, ep, deadline, pl[q]);
    if (!ok) break;
#pragma unroll
    for (int r = 0; r < kMaxAG; ++r)
      if (r == rank)
#pragma unroll
        for (int q = 0; q < 4; ++q) pl[q][r] = R.planes4[q * m + j];
    double wrap0 = 0.0, wrap1 = 0.0;  // w_{p-1}: the left neighbour of rank 0 (cyclic)
#pragma unroll
    for (int r = 0; r < kMaxAG; ++r)
      if (r == p - 1 && cyc) { wrap0 = pl[2][r]; wrap1 = pl[3][r]; }
    double xa0 = 0.0, xa1 = 0.0, xn0 = 0.0, xn1 = 0.0;
    const double* gi = R.ainv + (size_t)(2 * rank) * 2 * p;
    const double* gn = R.ainv + (size_t)(2 * (nx < 0 ? 0 : nx)) * 2 * p;
#pragma unroll
    for (int r = 0; r < kMaxAG; ++r) {
      if (r >= p) continue;
      const double b0 = pl[0][r] - (r > 0 ? pl[2][r > 0 ? r - 1 : 0] : wrap0);
      const double b1 = pl[1][r] - (r > 0 ? pl[3][r > 0 ? r - 1 : 0] : wrap1);
      xa0 += __ldg(gi + 2 * r) * b0 + __ldg(gi + 2 * r + 1) * b1;
      xa1 += __ldg(gi + 2 * p + 2 * r) * b0 + __ldg(gi + 2 * p + 2 * r + 1) * b1;
      xn0 += __ldg(gn + 2 * r) * b0 + __ldg(gn + 2 * r + 1) * b1;
      xn1 += __ldg(gn + 2 * p + 2 * r) * b0 + __ldg(gn + 2 * p + 2 * r + 1) * b1;
    }
    if (nx < 0) xn0 = xn1 = 0.0;
    const int64_t o = j / inner, cc = j - o * inner;
    R.x[o * n * inner + cc] = xa0;
    R.x[(o * n + 1) * inner + cc] = xa1;
    R.xnext[j] = xn0;
    R.xnext[m + j] = xn1;
  }
  if (!ok) *reinterpret_cast<volatile int*>(A.err) = 1;
  stamp(kTrYRecv);  // the single all-gather round
  stamp(kTrXRecv);
  __syncthreads();
  if (threadIdx.x == 0) R.epoch[slice] = ep;
  stamp(kTrEnd);
}

// Pentadiagonal (r = 2) reduced phase, pairwise (P:346 with 2x2 blocks, reading R20): the
// y round sends w = L~ y_i[last two] right, b^_i = c_i - w_{i-1}; then the steps of the block
// schedule (factor.h penta_reduced_schedule): b^_i <- W b^_i - C0 b^_{src0} - C1 b^_{src1} with
// 2x2 matrices -- block PCR stages (a single partner when i - s = i + s), the fold W = F_i, and
// for cyclic non-power-of-two p the detach / reattach steps of P:271 / P:294 -- and the x~ round
// from the right.  Every message is a 2-vector of LL words; R.step[] carries the partners,
// R.ppcr the matrices ([step][12]: W | C0 | C1).
__global__ void __launch_bounds__(kP2PThreads, 1)
    k_reduced_penta_pcr(const P2PArgs A) {
  if (A.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");  // launched early (PDL)
  const int r_local = blockIdx.x / A.nslices;
  const int slice = blockIdx.x - r_local * A.nslices;
  const P2PRank& R = A.rk[r_local];
  const int p = A.p, q = A.q, rank = R.rank;
  const int64_t m = A.m;
  const int64_t c0 = (int64_t)slice * A.slice_cols;
  const int64_t c1 = std::min<int64_t>(m, c0 + A.slice_cols);
  const uint32_t ep = R.epoch[slice] + 1u;
  const unsigned long long deadline = globaltimer() + A.deadline_ns;
  const int64_t copy_off = (int64_t)(ep & 1u) * A.copy_words;
  // copy: [y: 2 planes][step k: 2 slots x 2 planes][x: 2 planes] of 2m LL words
  auto OFF_Y = [&](int pl) -> int64_t { return (int64_t)pl * 2 * m; };
  auto OFF_S = [&](int k, int slot, int pl) -> int64_t { return (int64_t)(2 + 4 * k + 2 * slot + pl) * 2 * m; };
  auto OFF_X = [&](int pl) -> int64_t { return (int64_t)(2 + 4 * q + pl) * 2 * m; };
  const bool cyc = A.cyclic != 0;
  const int right = cyc ? (rank + 1) % p : (rank + 1 < p ? rank + 1 : -1);
  const int left = cyc ? (rank + p - 1) % p : (rank > 0 ? rank - 1 : -1);
  unsigned long long* const mine = R.mbox + copy_off;
  unsigned long long* tr = A.trace ? A.trace + (size_t)blockIdx.x * kP2PTrace : nullptr;
  auto stamp = [&](int k) {
    if (tr && threadIdx.x == 0) tr[k] = globaltimer();
  };
  stamp(kTrStart);
  bool ok = true;
  // the slice's columns in batches of kMaxCpt per thread (see k_reduced_p2p)
  for (int64_t cb0 = c0; cb0 < c1 && ok; cb0 += (int64_t)kP2PThreads * kMaxCpt) {
  const int64_t cb1 = std::min<int64_t>(c1, cb0 + (int64_t)kP2PThreads * kMaxCpt);
  double b0[kMaxCpt], b1[kMaxCpt];
  int64_t col[kMaxCpt];
  int nc = 0;
#pragma unroll
  for (int i = 0; i < kMaxCpt; ++i) {
    const int64_t j = cb0 + threadIdx.x + (int64_t)i * kP2PThreads;
    col[i] = j;
    if (j < cb1) nc = i + 1;
  }
  // receive the 2-vectors of `nc` columns from mailbox offsets o0 / o1 (batched sweep)
  auto recv2 = [&](int64_t o0, int64_t o1, double (&v0)[kMaxCpt], double (&v1)[kMaxCpt]) {
    uint32_t pend = 0;
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i)
      if (i < nc) pend |= 3u << (2 * i);
    int spins = 0;
    while (pend && ok) {
      unsigned long long w0[2 * kMaxCpt], w1[2 * kMaxCpt];
#pragma unroll
      for (int k = 0; k < 2 * kMaxCpt; ++k)
        if (pend & (1u << k)) dev::ll_load(mine + ((k & 1) ? o1 : o0) + 2 * col[k >> 1], &w0[k], &w1[k]);
#pragma unroll
      for (int k = 0; k < 2 * kMaxCpt; ++k)
        if ((pend & (1u << k)) && dev::ll_ready(w0[k], w1[k], ep)) {
          const double v = dev::ll_value(w0[k], w1[k]);
          if (k & 1) v1[k >> 1] = v;
          else v0[k >> 1] = v;
          pend &= ~(1u << k);
        }
      if (pend && ++spins == 64) {
        spins = 0;
        if (globaltimer() > deadline) ok = false;
      }
    }
  };
  // ---- (a2) w_i = L~ y_i[last two] -> right neighbour; b^_i = c_i - w_{i-1} ----
  // (the planes are loaded before the first LL store: the stores are asm volatile with a memory
  // clobber, a load between two of them would serialise the HBM latencies)
  double pw0[kMaxCpt], pw1[kMaxCpt], pc0[kMaxCpt], pc1[kMaxCpt];
#pragma unroll
  for (int i = 0; i < kMaxCpt; ++i) {
    pw0[i] = pw1[i] = pc0[i] = pc1[i] = 0.0;
    if (i < nc) {
      pc0[i] = R.planes4[col[i]];
      pc1[i] = R.planes4[R.pstride + col[i]];
      pw0[i] = R.planes4[2 * R.pstride + col[i]];
      pw1[i] = R.planes4[3 * R.pstride + col[i]];
    }
  }
  if (right >= 0) {
    unsigned long long* dst = R.peer_mbox[right] + copy_off;
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i)
      if (i < nc) {
        dev::ll_store(dst + OFF_Y(0) + 2 * col[i], pw0[i], ep);
        dev::ll_store(dst + OFF_Y(1) + 2 * col[i], pw1[i], ep);
      }
  }
  stamp(kTrYSent);
  {
    double w0[kMaxCpt], w1[kMaxCpt];
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i) w0[i] = w1[i] = 0.0;
    if (left >= 0) recv2(OFF_Y(0), OFF_Y(1), w0, w1);
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i)
      if (i < nc) {
        b0[i] = pc0[i] - w0[i];
        b1[i] = pc1[i] - w1[i];
      }
  }
  stamp(kTrYRecv);
  // ---- (a3) block PCR steps ----
  for (int st = 0; st < q && ok; ++st) {
    const P2PStep& S = R.step[st];
    for (int d = 0; d < 2; ++d) {
      const int dst = d ? S.dst1 : S.dst0, slot = d ? S.dslot1 : S.dslot0;
      if (dst < 0) continue;
      unsigned long long* dp = R.peer_mbox[dst] + copy_off;
#pragma unroll
      for (int i = 0; i < kMaxCpt; ++i)
        if (i < nc) {
          dev::ll_store(dp + OFF_S(st, slot, 0) + 2 * col[i], b0[i], ep);
          dev::ll_store(dp + OFF_S(st, slot, 1) + 2 * col[i], b1[i], ep);
        }
    }
    double u0[kMaxCpt], u1[kMaxCpt], v0[kMaxCpt], v1[kMaxCpt];
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i) u0[i] = u1[i] = v0[i] = v1[i] = 0.0;
    if (S.src0 >= 0) recv2(OFF_S(st, 0, 0), OFF_S(st, 0, 1), u0, u1);
    if (S.src1 >= 0) recv2(OFF_S(st, 1, 0), OFF_S(st, 1, 1), v0, v1);
    const double* M = R.ppcr + 12 * st;  // W | C0 | C1 (row-major 2x2)
    const double w00 = M[0], w01 = M[1], w10 = M[2], w11 = M[3];
    const double a00 = M[4], a01 = M[5], a10 = M[6], a11 = M[7];
    const double g00 = M[8], g01 = M[9], g10 = M[10], g11 = M[11];
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i)
      if (i < nc) {
        const double n0 = (w00 * b0[i] + w01 * b1[i]) - (a00 * u0[i] + a01 * u1[i]) - (g00 * v0[i] + g01 * v1[i]);
        const double n1 = (w10 * b0[i] + w11 * b1[i]) - (a10 * u0[i] + a11 * u1[i]) - (g10 * v0[i] + g11 * v1[i]);
        b0[i] = n0;
        b1[i] = n1;
      }
    stamp(kTrStep0 + st);
  }
  // (the fold x~_i = F_i b^_i and the reattach steps are steps of the schedule)
  // ---- (a4) x~_i -> left neighbour; x~_{i+1} from the right ----
  if (ok && left >= 0) {
    unsigned long long* dst = R.peer_mbox[left] + copy_off;
#pragma unroll
    for (int i = 0; i < kMaxCpt; ++i)
      if (i < nc) {
        dev::ll_store(dst + OFF_X(0) + 2 * col[i], b0[i], ep);
        dev::ll_store(dst + OFF_X(1) + 2 * col[i], b1[i], ep);
      }
  }
  double xn0[kMaxCpt], xn1[kMaxCpt];
#pragma unroll
  for (int i = 0; i < kMaxCpt; ++i) xn0[i] = xn1[i] = 0.0;
  if (ok && right >= 0) recv2(OFF_X(0), OFF_X(1), xn0, xn1);
  stamp(kTrXRecv);
  if (!ok) *reinterpret_cast<volatile int*>(A.err) = 1;
  const int64_t n = A.lay.n, inner = A.lay.inner;
#pragma unroll
  for (int i = 0; i < kMaxCpt; ++i)
    if (i < nc) {
      const int64_t j = col[i];
      const int64_t o = j / inner, cc = j - o * inner;
      R.x[o * n * inner + cc] = b0[i];
      R.x[(o * n + 1) * inner + cc] = b1[i];
      R.xnext[j] = xn0[i];
      R.xnext[m + j] = xn1[i];
    }
  }  // column batches
  __syncthreads();
  if (threadIdx.x == 0) R.epoch[slice] = ep;
  if (tr) stamp(kTrEnd);
}

cudaError_t launch_reduced_penta_pcr(const P2PArgs& A, int nranks_launch, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(A.nslices * nranks_launch), 1, 1);
  cfg.blockDim = dim3(kP2PThreads, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (nranks_launch > 1) {
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.numAttrs = 1;
  } else if (A.pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 1;
  }
  cfg.attrs = attr;
  return cudaLaunchKernelEx(&cfg, k_reduced_penta_pcr, A);
}

cudaError_t launch_reduced_allgather_r2(const P2PArgs& A, int nranks_launch, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(A.nslices * nranks_launch), 1, 1);
  cfg.blockDim = dim3(kP2PThreads, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = nranks_launch > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_reduced_allgather_r2, A);
}

cudaError_t launch_reduced_p2p(const P2PArgs& A, int nranks_launch, cudaStream_t s, int nrows) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(A.nslices * std::max(nranks_launch, nrows)), 1, 1);
  cfg.blockDim = dim3(kP2PThreads, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (nranks_launch > 1) {  // loopback: all CTAs co-resident (they wait on each other)
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.numAttrs = 1;
  } else if (A.pdl) {  // one rank per launch: staged while the tile kernel drains (PDL)
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 1;
  }
  cfg.attrs = attr;
  return A.allgather ? cudaLaunchKernelEx(&cfg, k_reduced_allgather, A)
                     : cudaLaunchKernelEx(&cfg, k_reduced_p2p, A);
}

int p2p_slices(int64_t m, int nranks_launch, int num_sms, int kind) {
  // one wave: <= resident CTAs in total (the schedule kernels batch wider slices)
  const void* fn = kind == 0 ? (const void*)k_reduced_p2p
                 : kind == 1 ? (const void*)k_reduced_allgather
                 : kind == 2 ? (const void*)k_reduced_allgather_r2 : (const void*)k_reduced_penta_pcr;
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kP2PThreads, 0) !=
          cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    per_sm = 1;
  }
  const int64_t cap = std::max<int64_t>(1, (int64_t)per_sm * num_sms / nranks_launch);
  int64_t ns = std::min<int64_t>(cap, (m + kP2PThreads - 1) / kP2PThreads);
  // one wave of co-resident CTAs always (rows of one GPU wait on each other); the schedule
  // kernels loop over batches of kMaxCpt columns per thread when a slice is wider
  return (int)std::max<int64_t>(1, ns);
}

// one epoch copy: [2 + 2q slots][2m LL words] (schedule) or [2 planes][p sources][2m] (all-gather)
int64_t p2p_copy_words(int64_t m, int q, int p, bool allgather, int planes) {
  return (int64_t)std::max(2 + 2 * q, allgather ? planes * p : 0) * 2 * m;
}
// [2 epoch copies][copy]  +  (derivative) [2 copies][4 halo rows][2m]
size_t p2p_mailbox_words(int64_t copy_words, int64_t m, bool halo) {
  return (size_t)2 * (size_t)copy_words + (halo ? (size_t)2 * 4 * 2 * (size_t)m : 0);
}

// (a0) halo of the compact-derivative stencil for nparts > 1: rows 0, 1 of this slab
// go to the left neighbour (its rows n, n+1) and rows n-2, n-1 to the right neighbour (its rows
// -2, -1), as LL words into their mailboxes; the incoming words become halo_lo / halo_hi.
__global__ void __launch_bounds__(kP2PThreads) k_halo_p2p(const P2PArgs A) {
  const int r_local = blockIdx.x / A.nslices;
  const int slice = blockIdx.x - r_local * A.nslices;
  const P2PRank& R = A.rk[r_local];
  const int p = A.p, rank = R.rank;
  const int64_t m = A.m, n = A.lay.n, inner = A.lay.inner;
  // R.mbox / R.peer_mbox point at the halo region of the mailboxes and R.epoch at the halo's
  // own per-slice epochs: the reduced-phase kernels keep theirs, so each exchange keeps its
  // epoch-parity double buffering (a derivative solve advances each counter by exactly one)
  const uint32_t ep = R.epoch[slice] + 1u;
  const unsigned long long deadline = globaltimer() + A.deadline_ns;
  const int64_t hoff = (int64_t)(ep & 1u) * 8 * m;
  const int left = (rank + p - 1) % p, right = (rank + 1) % p;
  const int64_t c0 = (int64_t)slice * A.slice_cols;
  const int64_t c1 = std::min<int64_t>(m, c0 + A.slice_cols);
  bool ok = true;
  // kHU columns per thread and pass: every f row load is issued before the first LL store (the
  // stores are asm volatile with a memory clobber: a load per store would serialise HBM
  // latencies), and every pending word of the receive is loaded before any is tested
  constexpr int kHU = 4;
  unsigned long long* lo = R.peer_mbox[right] + hoff;  // right neighbour's rows -2, -1
  unsigned long long* hi = R.peer_mbox[left] + hoff;   // left neighbour's rows n, n+1
  for (int64_t jb = c0 + threadIdx.x; jb < c1; jb += (int64_t)kP2PThreads * kHU) {
    double v[kHU][4];
#pragma unroll
    for (int u = 0; u < kHU; ++u) {
      const int64_t j = jb + (int64_t)u * kP2PThreads;
      if (j >= c1) continue;
      const int64_t o = j / inner, c = j - o * inner;
      const double* fc = R.f + o * n * inner + c;
      v[u][0] = fc[(n - 2) * inner];
      v[u][1] = fc[(n - 1) * inner];
      v[u][2] = fc[0];
      v[u][3] = fc[inner];
    }
#pragma unroll
    for (int u = 0; u < kHU; ++u) {
      const int64_t j = jb + (int64_t)u * kP2PThreads;
      if (j >= c1) continue;
      ll_send(lo + 2 * j, v[u][0], ep);
      ll_send(lo + 2 * m + 2 * j, v[u][1], ep);
      ll_send(hi + 4 * m + 2 * j, v[u][2], ep);
      ll_send(hi + 6 * m + 2 * j, v[u][3], ep);
    }
  }
  const unsigned long long* mine = R.mbox + hoff;
  for (int64_t jb = c0 + threadIdx.x; jb < c1 && ok; jb += (int64_t)kP2PThreads * kHU) {
    double v[kHU][4];
    uint32_t pend = 0;
#pragma unroll
    for (int u = 0; u < kHU; ++u)
      if (jb + (int64_t)u * kP2PThreads < c1) pend |= 0xfu << (4 * u);
    int spins = 0;
    while (pend && ok) {
      unsigned long long w0[4 * kHU], w1[4 * kHU];
#pragma unroll
      for (int k = 0; k < 4 * kHU; ++k)
        if (pend & (1u << k))
          dev::ll_load(mine + (int64_t)(k & 3) * 2 * m + 2 * (jb + (int64_t)(k >> 2) * kP2PThreads), &w0[k], &w1[k]);
#pragma unroll
      for (int k = 0; k < 4 * kHU; ++k)
        if ((pend & (1u << k)) && dev::ll_ready(w0[k], w1[k], ep)) {
          v[k >> 2][k & 3] = dev::ll_value(w0[k], w1[k]);
          pend &= ~(1u << k);
        }
      if (pend && ++spins == 64) {
        spins = 0;
        if (globaltimer() > deadline) ok = false;
      }
    }
    if (!ok) break;
#pragma unroll
    for (int u = 0; u < kHU; ++u) {
      const int64_t j = jb + (int64_t)u * kP2PThreads;
      if (j >= c1) continue;
      R.halo_lo[j] = v[u][0];
      R.halo_lo[m + j] = v[u][1];
      R.halo_hi[j] = v[u][2];
      R.halo_hi[m + j] = v[u][3];
    }
  }
  if (!ok) *reinterpret_cast<volatile int*>(A.err) = 2;
  __syncthreads();
  if (threadIdx.x == 0) R.epoch[slice] = ep;
}

cudaError_t launch_halo_p2p(const P2PArgs& A, int nranks_launch, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(A.nslices * nranks_launch), 1, 1);
  cfg.blockDim = dim3(kP2PThreads, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = nranks_launch > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_halo_p2p, A);
}

}  // namespace ctri
