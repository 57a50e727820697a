// capi.cu -- implementation of include/ctri.h: plan creation (pre-factorisation),
// the per-solve phase sequence (a1)-(a4) with NCCL (or test-only loopback) exchanges,
// the compact-derivative entry point and the statistics / host-query functions.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "internal.h"

using namespace ctri;

namespace {
thread_local std::string g_err;

ctri_status fail(ctri_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? CTRI_ERR_OOM : CTRI_ERR_CUDA,         \
                  std::string(#expr) + ": " + cudaGetErrorString(e_));                    \
  } while (0)

#define NCCL_TRY(expr)                                                                    \
  do {                                                                                    \
    ncclResult_t r_ = (expr);                                                             \
    if (r_ != ncclSuccess)                                                                \
      return fail(CTRI_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_));     \
  } while (0)

#define TRY(expr)                      \
  do {                                 \
    ctri_status s_ = (expr);           \
    if (s_ != CTRI_OK) return s_;      \
  } while (0)

// timing event slots
enum { EV_START = 0, EV_LOCAL, EV_YX, EV_BHAT, EV_STAGE0, EV_XX = EV_STAGE0 + CTRI_MAX_STAGES,
       EV_BACK, EV_COUNT };

ctri_status upload(double** dst, const std::vector<double>& src, cudaStream_t s) {
  CUDA_TRY(cudaMalloc(dst, std::max<size_t>(1, src.size()) * sizeof(double)));
  if (!src.empty())
    CUDA_TRY(cudaMemcpyAsync(*dst, src.data(), src.size() * sizeof(double),
                             cudaMemcpyHostToDevice, s));
  return CTRI_OK;
}

ctri_status alloc_plane(double** p, int64_t count) {
  CUDA_TRY(cudaMalloc(p, std::max<int64_t>(1, count) * sizeof(double)));
  CUDA_TRY(cudaMemset(*p, 0, std::max<int64_t>(1, count) * sizeof(double)));
  return CTRI_OK;
}

// The P2P deadline word lives in mapped pinned host memory: kernels store to it over the bus
// only on failure, and the host reads it at the next call without synchronising.
ctri_status alloc_err(Plan* P) {
  CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&P->h_err), sizeof(int), cudaHostAllocMapped));
  *reinterpret_cast<volatile int*>(P->h_err) = 0;
  CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&P->d_err), P->h_err, 0));
  return CTRI_OK;
}

// A plan whose P2P wait hit its deadline is out of step with its peers (epochs, mailboxes):
// every later call fails instead of returning silently wrong results.
ctri_status check_poisoned(const std::vector<Plan*>& G) {
  for (const Plan* P : G)
    if (P->h_err && *reinterpret_cast<volatile int*>(P->h_err))
      return fail(CTRI_ERR_CUDA, "a previous solve timed out waiting for a peer (device deadline, "
                                 "error word " + std::to_string(*reinterpret_cast<volatile int*>(P->h_err)) +
                                 "); the plan is unusable: destroy it");
  return CTRI_OK;
}

void free_plan(Plan* P) {
  if (!P) return;
  double* bufs[] = {P->d_cp,    P->d_inv_den, P->d_S,      P->d_R,       P->d_vS,    P->d_vR,
                    P->yf,      P->yl,
                    P->bt,      P->yl_prev,   P->bh,       P->recv_m,    P->recv_p,  P->xt,
                    P->xt_next, P->halo_lo,   /* halo_hi: inside halo_lo */ P->send_lo, P->send_hi, P->tile.d_pcr,
                    P->d_stage_b, P->d_stage_x, P->d_plu,    P->d_pSR,     P->d_ainv,  P->d_planes4,
                    P->d_xnext2, P->d_ppcr, P->d_vppcr, P->ptc.d_tab};
  for (double* b : bufs)
    if (b) cudaFree(b);
  for (cudaEvent_t e : P->ev) cudaEventDestroy(e);
  for (size_t r = 0; r < P->peer_alloc.size(); ++r)
    if (r < P->peer_ipc.size() && P->peer_ipc[r] && P->peer_alloc[r]) cudaIpcCloseMemHandle(P->peer_alloc[r]);
  if (P->mbox_alloc) cudaFree(P->mbox_alloc);
  if (P->h_err) cudaFreeHost(P->h_err);
  if (P->d_epoch) cudaFree(P->d_epoch);
  if (P->d_hepoch) cudaFree(P->d_hepoch);
  if (P->d_trace) cudaFree(P->d_trace);
  if (P->d_fctr) cudaFree(P->d_fctr);
  if (P->e2e_sub) free_plan(P->e2e_sub);
  for (cudaEvent_t e : P->e2e_ev) cudaEventDestroy(e);
  if (P->e2e_h2d) cudaStreamDestroy(P->e2e_h2d);
  if (P->e2e_d2h) cudaStreamDestroy(P->e2e_d2h);
  if (P->comm) ncclCommDestroy(P->comm);
  delete P;
}

bool has_left(const Plan& P) { return P.cyclic || P.rank > 0; }
bool has_right(const Plan& P) { return P.cyclic || P.rank < P.p - 1; }
int wrap(const Plan& P, int r) { return ((r % P.p) + P.p) % P.p; }

// Common plan set-up (no communicator).
ctri_status plan_init(Plan* P, const int64_t gd[3], int sd, int p, int rank, const double bands[3],
                      int cyclic, uint32_t flags, cudaStream_t s) {
  if (!gd || !bands) return fail(CTRI_ERR_INVALID_ARG, "NULL dims or bands");
  if (sd < 0 || sd > 2) return fail(CTRI_ERR_INVALID_ARG, "solve_dim must be 0, 1 or 2");
  for (int k = 0; k < 3; ++k)
    if (gd[k] < 1) return fail(CTRI_ERR_INVALID_ARG, "global dims must be >= 1");
  if (p < 1 || rank < 0 || rank >= p) return fail(CTRI_ERR_INVALID_ARG, "bad nparts/rank");
  for (int k = 0; k < 3; ++k)
    if (!std::isfinite(bands[k])) return fail(CTRI_ERR_INVALID_ARG, "bands must be finite");
  if (gd[sd] % p != 0)
    return fail(CTRI_ERR_PARTITION_TOO_SMALL, "N is not divisible by nparts (equal split, P:5)");
  const int64_t n = gd[sd] / p;
  if (n < 3) return fail(CTRI_ERR_PARTITION_TOO_SMALL, "n = N/nparts < 3 (N_i = n-1 >= 2r)");
  if (cyclic && !is_pow2(p) && (p > kMaxP2PRanks || (flags & CTRI_FLAG_NCCL_ROUNDS)))
    return fail(CTRI_ERR_UNSUPPORTED,
                "cyclic non-power-of-two nparts: detach/reattach (P:271) runs in the fused P2P path "
                "only (nparts <= 16, without CTRI_FLAG_NCCL_ROUNDS)");
  std::memcpy(P->gdims, gd, sizeof(P->gdims));
  P->sd = sd;
  P->p = p;
  P->rank = rank;
  P->cyclic = cyclic ? 1 : 0;
  P->flags = flags;
  P->bands = Bands{bands[0], bands[1], bands[2]};
  P->lay.n = n;
  P->lay.outer = 1;
  P->lay.inner = 1;
  for (int k = 0; k < sd; ++k) P->lay.outer *= gd[k];
  for (int k = sd + 1; k < 3; ++k) P->lay.inner *= gd[k];
  CUDA_TRY(cudaGetDevice(&P->device));
  CUDA_TRY(cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, P->device));

  // virtual partitions (nparts == 1): the slab is solved as vp partitions of n/vp rows so the
  // local-solve clusters are small enough to occupy every GPC
  // test knobs of the P2P deadline path, read once per plan (never on the solve path)
  if (const char* e = std::getenv("CTRI_TEST_P2P_DEADLINE_MS"))
    if (*e) P->deadline_ns = (unsigned long long)std::max(1, std::atoi(e)) * 1000000ull;
  if (const char* e = std::getenv("CTRI_TEST_P2P_DROP_RANK"))
    if (*e) P->test_drop_rank = std::atoi(e);
  P->vp = 1;
  const char* vp_env = std::getenv("CTRI_VPARTS");  // measurement knob (any axis)
  if (vp_env && !*vp_env) vp_env = nullptr;        // set but empty: default rule
  if (p == 1 && !(flags & CTRI_FLAG_DERIV) && (P->lay.inner >= 16 || P->lay.inner == 1 || vp_env)) {
    // measured: virtual slabs of 1024 rows (clusters of 4) are fastest for n >= 4096 on a
    // strided axis; 2048 rows (clusters of 2, 4 partitions at n = 8192) on the contiguous axis
    int want = n >= 4096 ? (int)std::min<int64_t>(P->lay.inner == 1 ? 4 : 8,
                                                  n / (P->lay.inner == 1 ? 2048 : 1024))
                         : 1;
    if (vp_env) want = std::atoi(vp_env);
    if (want > 1 && want <= 8 && is_pow2(want) && n % want == 0 && n / want >= 512 &&
        (vp_env || is_pow2(n / want))) {
      P->vp = want;
    } else if (!vp_env && want > 1 && P->lay.inner >= 16) {
      // n not a power-of-two multiple of 1024 (e.g. 6144): the most partitions (<= 8) whose
      // length is a power of two the tile kernel takes; their reduced system (vp not a power of
      // two) is solved with a plan-time dense inverse in k_reduced_local, without the chain
      for (int w = std::min(want, 8); w > 1; --w)
        if (n % w == 0 && is_pow2(n / w) && n / w >= 512) {
          P->vp = w;
          break;
        }
    }
  }
  // nparts > 1: "virtual rows" -- every rank's slab is solved as vp partitions too and the
  // reduced system has nparts * vp rows, exchanged over the same LL P2P path (rows on the same
  // GPU exchange through its own mailbox).  Strided axis with outer == 1 (solve index 0): as
  // with one partition, partitions of 1024 rows (measured cfg2: N = 2 0.967 -> 0.890 ms with
  // vp = 4, N = 4 0.478 -> 0.466 ms with vp = 2).
  if (p > 1 && !(flags & (CTRI_FLAG_DERIV | CTRI_FLAG_NCCL_ROUNDS | CTRI_FLAG_ALLGATHER |
                          CTRI_FLAG_FUSED_REDUCED)) &&
      P->lay.outer == 1 && P->lay.inner >= 16) {
    int want = n >= 2048 ? (int)std::min<int64_t>(8, n / 1024) : 1;
    while (want > 1 && p * want > kMaxP2PRanks) want /= 2;
    if (vp_env) want = std::atoi(vp_env);
    // (the knob may go down to 16-row partitions: tests use them to make the reduced couplings
    // between virtual rows large enough to see)
    if (want > 1 && want <= 8 && is_pow2(want) && n % want == 0 && n / want >= (vp_env ? 16 : 512) &&
        p * want <= kMaxP2PRanks)
      P->vp = want;
  }
  P->tlay = P->lay;
  P->tlay.outer = P->lay.outer * P->vp;
  P->tlay.n = n / P->vp;
  const int64_t nv = P->tlay.n;

  // ---- pre-factorisation ----
  FactorError fe;
  // the (virtual) partition the local kernels solve: nv - 1 interior rows
  if (!partition_factor(nv - 1, P->bands, &P->vpart, &fe)) return fail((ctri_status)fe.code, fe.detail);
  P->vwindow = backsub_window(P->vpart);
  P->window = P->vwindow;  // tile_configure's checks (the fused layout needs vp == 1: same level)
  std::string why;
  const bool tile_ok = tile_configure(*P, &why);
  // virtual partitions finish (a2)-(a4) inside the tile kernel when its configuration allows
  // (the virtual-partition chain).  With nparts > 1 that makes two levels: the chain computes
  // D_i^{-1} b_i of the whole slab (its internal interfaces solved on chip), and the reduced
  // system across the GPUs keeps the paper's one row per rank.
  // (two levels are opt-in, CTRI_TWO_LEVEL=1: measured on 2 and 4 B200s the in-kernel window
  // work cost more than the virtual rows' window pass it saves -- DESIGN.md section 5)
  P->vchain = tile_ok && !P->tile.contig && P->vp > 1 && is_pow2(P->vp) && P->tile.vc_ok && !knob_no_vchain() &&
              !knob_copy_only() && (p == 1 || knob_two_level());
  P->rvp = (p > 1 && P->vchain) ? 1 : P->vp;
  const int64_t rn = n / P->rvp;  // rows per reduced-system row's partition
  const int pr = p * P->rvp;      // rows of the reduced system (virtual rows included)
  if (P->rvp == P->vp) {
    P->part = P->vpart;
  } else if (!partition_factor(rn - 1, P->bands, &P->part, &fe)) {
    return fail((ctri_status)fe.code, fe.detail);
  }
  const Partition& pt = P->part;
  const int64_t last = rn - 2;
  std::vector<double> L(pr), D(pr), U(pr);
  for (int i = 0; i < pr; ++i) {
    const bool lft = cyclic || i > 0, rgt = cyclic || i < pr - 1;
    L[i] = lft ? -P->bands.l * pt.S[last] : 0.0;                                 // Eq. Li_hat
    D[i] = P->bands.d - (lft ? P->bands.l * pt.R[last] : 0.0) - P->bands.u * pt.S[0];  // Eq. Di_hat
    U[i] = rgt ? -P->bands.u * pt.R[0] : 0.0;                                    // Eq. Ui_hat
  }
  // reduced-system schedule (PCR, or detach/PCR/fold/reattach for cyclic non-power-of-two p)
  if (!reduced_schedule(pr, cyclic != 0, L, D, U, pivot_threshold(P->bands), &P->sched, &fe))
    return fail((ctri_status)fe.code, fe.detail);
  if ((int)P->sched.steps.size() > kMaxP2PSteps)
    return fail(CTRI_ERR_UNSUPPORTED, "reduced-system schedule too long");
  if (!cyclic || is_pow2(pr)) {  // stride-PCR multipliers for the NCCL-rounds / local kernels
    if (!pcr_factor(pr, cyclic != 0, L, D, U, pivot_threshold(P->bands), &P->gpcr, &fe))
      return fail((ctri_status)fe.code, fe.detail);
  } else {
    P->gpcr = PcrTables();
    P->gpcr.P = pr;
    P->gpcr.stages = P->sched.pcr_stages;
    P->gpcr.inv.assign(pr, 0.0);
  }
  if (P->gpcr.stages > CTRI_MAX_STAGES) return fail(CTRI_ERR_UNSUPPORTED, "too many PCR stages");
  P->inv_closure = P->gpcr.inv[0];
  // one GPU, a cyclic vp-row system with vp not a power of two: k_reduced_local applies its
  // plan-time inverse (the reduced matrix of Eqs. Li_hat..Ui_hat, dense Gaussian elimination)
  if (p == 1 && P->vp > 1 && cyclic && !is_pow2(P->vp) &&
      !reduced_inverse(pr, true, L, D, U, pivot_threshold(P->bands), &P->ainv, &fe))
    return fail((ctri_status)fe.code, fe.detail);
  P->window = backsub_window(pt);
  // two levels: the slab's internal interfaces 1..vp-1 as an acyclic vp-row system whose row 0
  // (the GPU interface, not part of D_i) is decoupled: L^ = D^ - 1 = U^ = 0 there, no coupling
  // of row 1 to it nor of row vp-1 past the slab (Eqs. Li_hat..Ui_hat at the virtual level)
  if (p > 1 && P->vchain) {
    const Partition& vt = P->vpart;
    const int64_t vl = nv - 2;
    const int vp = P->vp;
    std::vector<double> Lv(vp), Dv(vp), Uv(vp);
    for (int v = 0; v < vp; ++v) {
      Lv[v] = v >= 2 ? -P->bands.l * vt.S[vl] : 0.0;
      Dv[v] = v == 0 ? 1.0 : P->bands.d - P->bands.l * vt.R[vl] - P->bands.u * vt.S[0];
      Uv[v] = (v >= 1 && v <= vp - 2) ? -P->bands.u * vt.R[0] : 0.0;
    }
    if (!pcr_factor(vp, false, Lv, Dv, Uv, pivot_threshold(P->bands), &P->vpcr, &fe))
      return fail((ctri_status)fe.code, fe.detail);
  }

  // ---- device tables ----
  TRY(upload(&P->d_S, pt.S, s));
  TRY(upload(&P->d_R, pt.R, s));
  if (P->rvp != P->vp) {  // the chain's own (virtual-level) S, R
    TRY(upload(&P->d_vS, P->vpart.S, s));
    TRY(upload(&P->d_vR, P->vpart.R, s));
  }
  const int64_t m = P->lay.m();
  if (tile_ok) {
    P->local_kernel = P->tile.contig ? 2 : 1;
    std::vector<double> t;
    t.insert(t.end(), P->tile.pcr.alpha.begin(), P->tile.pcr.alpha.end());
    t.insert(t.end(), P->tile.pcr.gamma.begin(), P->tile.pcr.gamma.end());
    t.insert(t.end(), P->tile.pcr.inv.begin(), P->tile.pcr.inv.end());
    TRY(upload(&P->tile.d_pcr, t, s));
  } else {
    P->local_kernel = 0;
    TRY(upload(&P->d_cp, P->vpart.th.cp, s));
    TRY(upload(&P->d_inv_den, P->vpart.th.inv_den, s));
  }
  if (p > 1 || P->vp > 1) {
    double** planes[] = {&P->yf, &P->yl, &P->bt, &P->yl_prev, &P->bh, &P->recv_m, &P->recv_p,
                         &P->xt, &P->xt_next};
    for (double** pl : planes) TRY(alloc_plane(pl, m * P->rvp));
  }
  if (flags & CTRI_FLAG_ALLGATHER) {
    if (p < 2 || p > kMaxAG || (flags & CTRI_FLAG_NCCL_ROUNDS))
      return fail(CTRI_ERR_UNSUPPORTED, "CTRI_FLAG_ALLGATHER needs 2 <= nparts <= 8 and the P2P path");
    if (!reduced_inverse(p, cyclic != 0, L, D, U, pivot_threshold(P->bands), &P->ainv, &fe))
      return fail((ctri_status)fe.code, fe.detail);
    P->allgather = true;
  }
  // (a2)-(a4) fused into the tile kernel (real GPUs; the loopback group cannot co-schedule one
  // kernel per rank): window rows stashed on chip, planes all-gathered as LL words
  P->fused = (flags & CTRI_FLAG_FUSED_REDUCED) && p > 1 && p <= 8 && !P->loopback &&
             P->local_kernel == 1 && P->tile.fused_ok &&
             !(flags & (CTRI_FLAG_NCCL_ROUNDS | CTRI_FLAG_FULL_BACKSUB | CTRI_FLAG_ALLGATHER));
  if (P->fused) {
    std::vector<double> inv;
    if (!reduced_inverse(p, cyclic != 0, L, D, U, pivot_threshold(P->bands), &inv, &fe))
      return fail((ctri_status)fe.code, fe.detail);
    const int nx = rank + 1;
    for (int r = 0; r < p; ++r) {
      P->fg0[r] = inv[(size_t)rank * p + r];
      P->fg1[r] = (nx < p || cyclic) ? inv[(size_t)(nx % p) * p + r] : 0.0;
    }
    CUDA_TRY(cudaMalloc(&P->d_fctr, 2 * sizeof(unsigned int)));
    CUDA_TRY(cudaMemsetAsync(P->d_fctr, 0, 2 * sizeof(unsigned int), s));
    P->p2p_off = (int64_t)8 * p * m;  // [2 copies][2 planes][p rows][m] LL words
  }
  if (p > 1 && p <= kMaxP2PRanks && !(flags & CTRI_FLAG_NCCL_ROUNDS)) {
    // device-initiated reduced phase: double-buffered mailbox + epoch flags
    const int q = (int)P->sched.steps.size();
    // one mailbox (two epoch copies) per virtual row of this rank
    P->p2p_nslices = p2p_slices(m, (P->loopback ? p : 1) * P->rvp, P->num_sms, P->allgather ? 1 : 0);
    P->p2p_vrow_words = 2 * p2p_copy_words(m, q, pr, P->allgather);
    P->mbox_bytes = sizeof(unsigned long long) *
                    ((size_t)P->p2p_off + (size_t)P->rvp * P->p2p_vrow_words +
                     ((flags & CTRI_FLAG_DERIV) ? p2p_mailbox_words(0, m, true) : 0));
    CUDA_TRY(cudaMalloc(&P->mbox_alloc, P->mbox_bytes));
    CUDA_TRY(cudaMemsetAsync(P->mbox_alloc, 0, P->mbox_bytes, s));
    TRY(alloc_err(P));
    CUDA_TRY(cudaMalloc(&P->d_epoch, sizeof(unsigned int) * P->p2p_nslices * P->rvp));
    CUDA_TRY(cudaMemsetAsync(P->d_epoch, 0, sizeof(unsigned int) * P->p2p_nslices * P->rvp, s));
    if (flags & CTRI_FLAG_DERIV) {  // the halo exchange: its own mailbox region and epochs
      P->halo_off = P->p2p_off + (int64_t)P->rvp * P->p2p_vrow_words;
      CUDA_TRY(cudaMalloc(&P->d_hepoch, sizeof(unsigned int) * P->p2p_nslices));
      CUDA_TRY(cudaMemsetAsync(P->d_hepoch, 0, sizeof(unsigned int) * P->p2p_nslices, s));
    }
    P->p2p = true;
  }
  if (flags & CTRI_FLAG_DERIV) {
    if (!cyclic) return fail(CTRI_ERR_INVALID_ARG, "CTRI_FLAG_DERIV needs a cyclic plan");
    // halo_lo | halo_hi as one [2][2][m] allocation: the tile kernel loads a column tile's
    // halo rows from it with one TMA map (rows 0, 1: the slab above; rows 2, 3: below)
    TRY(alloc_plane(&P->halo_lo, 4 * m));
    P->halo_hi = P->halo_lo + 2 * m;
    TRY(alloc_plane(&P->send_lo, 2 * m));
    TRY(alloc_plane(&P->send_hi, 2 * m));
  }
  if (flags & CTRI_FLAG_TIMING) {
    P->ev.resize(EV_COUNT);
    for (auto& e : P->ev) CUDA_TRY(cudaEventCreate(&e));
  }
  // launches per solve
  int launches = 1;
  if (p > 1 && !P->fused) launches += P->p2p ? 2 /*reduced + window*/ : 1 /*bhat*/ + P->gpcr.stages + 1 /*backsub*/;
  if (p == 1 && P->vp > 1 && !P->vchain) launches += 2;  // local reduced system; window pass
  P->launches_per_solve = launches;
  CUDA_TRY(cudaStreamSynchronize(s));
  return CTRI_OK;
}

// Pentadiagonal plan (r = 2, penta.cu): validation, tables, P2P mailbox.
ctri_status penta_init(Plan* P, const int64_t gd[3], int sd, int p, int rank, const double bands[5],
                       int cyclic, uint32_t flags, cudaStream_t s) {
  if (!gd || !bands) return fail(CTRI_ERR_INVALID_ARG, "NULL dims or bands");
  if (sd < 0 || sd > 2) return fail(CTRI_ERR_INVALID_ARG, "solve_dim must be 0, 1 or 2");
  for (int k = 0; k < 3; ++k)
    if (gd[k] < 1) return fail(CTRI_ERR_INVALID_ARG, "global dims must be >= 1");
  if (p < 1 || rank < 0 || rank >= p) return fail(CTRI_ERR_INVALID_ARG, "bad nparts/rank");
  for (int k = 0; k < 5; ++k)
    if (!std::isfinite(bands[k])) return fail(CTRI_ERR_INVALID_ARG, "bands must be finite");
  if (gd[sd] % p != 0)
    return fail(CTRI_ERR_PARTITION_TOO_SMALL, "N is not divisible by nparts (equal split, P:5)");
  const int64_t n = gd[sd] / p;
  if (n < 6) return fail(CTRI_ERR_PARTITION_TOO_SMALL, "pentadiagonal: n = N/nparts < 6 (N_i = n-2 >= 4)");
  if (p > kMaxAG) return fail(CTRI_ERR_UNSUPPORTED, "pentadiagonal: nparts <= 8 (all-gather reduced solve)");
  if (flags & (CTRI_FLAG_NCCL_ROUNDS | CTRI_FLAG_DERIV | CTRI_FLAG_GENERIC_LOCAL))
    return fail(CTRI_ERR_UNSUPPORTED, "pentadiagonal plans: P2P all-gather path only, no derivative");
  std::memcpy(P->gdims, gd, sizeof(P->gdims));
  P->sd = sd;
  P->p = p;
  P->rank = rank;
  P->cyclic = cyclic ? 1 : 0;
  P->flags = flags;
  P->r = 2;
  std::memcpy(P->bands5, bands, sizeof(P->bands5));
  P->bands = Bands{bands[1], bands[2], bands[3]};
  P->lay.n = n;
  P->lay.outer = 1;
  P->lay.inner = 1;
  for (int k = 0; k < sd; ++k) P->lay.outer *= gd[k];
  for (int k = sd + 1; k < 3; ++k) P->lay.inner *= gd[k];
  // on-chip local solve (ptile.cu) where its geometry fits: one partition of 256..2048 rows, or
  // with one GPU and a longer strided slab the paper's partition method with vp = n / 1024
  // partitions on this GPU (reduced 2x2-block system over them, then the window pass).
  // Measured on the cfg2 grid: 1024-row partitions (clusters of 4, shuffle PCR) 2.32 ms,
  // 2048-row ones (clusters of 8, shared-memory PCR, half the window rows) 2.50 ms.
  // nparts > 1 (solve index 0, outer == 1): the same 1024-row partitions as "virtual rows" --
  // the reduced 2x2-block system has nparts * vp block rows, exchanged over the LL P2P path
  // (rows of one GPU through its own mailbox), as for the tridiagonal solve.  CTRI_VPARTS
  // overrides the count (measurement and test knob; 1: the slab as one partition).
  P->vp = 1;
  const bool vp_fit = P->lay.inner >= 32 && n > 1024 && n % 1024 == 0 && n / 1024 <= 8 &&
                      is_pow2(n / 1024) && !knob_penta_serial();
  if (vp_fit && (p == 1 || (P->lay.outer == 1 && !(flags & CTRI_FLAG_ALLGATHER) &&
                            p * (n / 1024) <= kMaxP2PRanks)))
    P->vp = (int)(n / 1024);
  if (p == 1 && P->vp == 1 && !vp_fit && P->lay.inner >= 32 && n > 2048 && !knob_penta_serial())
    for (int w = 8; w > 1; --w)  // e.g. 6144 = 6 x 1024: power-of-two partitions, dense reduced solve
      if (n % w == 0 && is_pow2(n / w) && n / w >= 256 && n / w <= 2048) {
        P->vp = w;
        break;
      }
  if (const char* e = std::getenv("CTRI_VPARTS"))
    if (*e && P->vp > 1) {
      const int want = std::atoi(e);
      if (want >= 1 && want <= P->vp && is_pow2(want)) P->vp = want;
    }
  P->rvp = p > 1 ? P->vp : 1;
  P->tlay = P->lay;
  P->tlay.outer = P->lay.outer * P->vp;
  P->tlay.n = n / P->vp;
  P->local_kernel = 3;
  CUDA_TRY(cudaGetDevice(&P->device));
  CUDA_TRY(cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, P->device));
  std::string why;
  ctri_status st = penta_plan_tables(P, s, &why);
  if (st != CTRI_OK) return fail(st, "pentadiagonal tables: " + why);
  if (!knob_penta_serial() && ptile_configure(*P, &why)) {
    P->local_kernel = 4;
    if ((st = upload(&P->ptc.d_tab, P->ptc.tab, s)) != CTRI_OK) return fail(st, "penta tile tables");
  } else if (P->vp > 1) {  // no on-chip solve: the slab as one partition, column-serial
    P->vp = 1;
    P->rvp = 1;
    P->tlay = P->lay;
    if ((st = penta_plan_tables(P, s, &why)) != CTRI_OK) return fail(st, "pentadiagonal tables: " + why);
  }
  const int64_t m = P->lay.m();
  if (p > 1) {
    // the 2x2-block step schedule (P:346 in block form; detach / PCR / fold / reattach for
    // cyclic non-power-of-two p, P:271 / P:294), or with CTRI_FLAG_ALLGATHER the one-round
    // all-gather (R20)
    P->ppcr = !(flags & CTRI_FLAG_ALLGATHER);
    int64_t copy_words = p2p_copy_words(m, 0, p, true, 4);
    if (P->ppcr) {
      double mx = 0;
      for (int k = 0; k < 5; ++k) mx = std::max(mx, std::fabs(bands[k]));
      BlockSchedule sc;
      FactorError fe;
      const int pr = p * P->rvp;  // block rows of the reduced system (virtual rows included)
      if (!penta_reduced_schedule(pr, cyclic != 0, P->pt, 1e-13 * mx, &sc, &fe))
        return fail((ctri_status)fe.code, fe.detail);
      const int q = (int)sc.steps.size();
      if (q > kMaxP2PSteps) return fail(CTRI_ERR_UNSUPPORTED, "pentadiagonal reduced schedule too long");
      P->ppcr_steps = q;
      P->sched.pcr_stages = sc.pcr_stages;  // (counts reported by ctri_get_stats)
      P->sched.detach_stages = sc.detach_stages;
      P->sched.detached_rows = sc.detached_rows;
      std::vector<double> tab;  // [virtual row][step][12]: W | C0 | C1 of this rank's rows
      P->pstep.assign((size_t)P->rvp * kMaxP2PSteps, P2PStep{1.0, 0.0, 0.0, -1, -1, -1, -1, 0, 0});
      for (int v = 0; v < P->rvp; ++v) {
        const int g = rank * P->rvp + v;  // global block row
        for (int k = 0; k < q; ++k) {
          const BlockSchedEntry& e = sc.steps[k][g];
          tab.insert(tab.end(), e.W, e.W + 4);
          tab.insert(tab.end(), e.C[0], e.C[0] + 4);
          tab.insert(tab.end(), e.C[1], e.C[1] + 4);
          P2PStep& stp = P->pstep[(size_t)v * kMaxP2PSteps + k];
          stp.src0 = (int8_t)e.src[0];
          stp.src1 = (int8_t)e.src[1];
          int nd = 0;  // this row's pre-step value goes to every row that reads it
          for (int r = 0; r < pr; ++r)
            for (int sl = 0; sl < 2; ++sl)
              if (sc.steps[k][r].src[sl] == g) {
                if (nd == 0) { stp.dst0 = (int8_t)r; stp.dslot0 = (int8_t)sl; }
                else if (nd == 1) { stp.dst1 = (int8_t)r; stp.dslot1 = (int8_t)sl; }
                ++nd;
              }
          if (nd > 2) return fail(CTRI_ERR_UNSUPPORTED, "pentadiagonal reduced schedule: > 2 readers");
        }
      }
      CUDA_TRY(cudaMalloc(&P->d_ppcr, sizeof(double) * tab.size()));
      CUDA_TRY(cudaMemcpyAsync(P->d_ppcr, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice, s));
      copy_words = (int64_t)(4 + 4 * q) * 2 * m;
    }
    P->p2p_nslices = p2p_slices(m, (P->loopback ? p : 1) * P->rvp, P->num_sms, P->ppcr ? 3 : 2);
    P->p2p_copy = copy_words;
    // one mailbox (two epoch copies) per virtual row of this rank
    P->p2p_off = 0;
    P->p2p_vrow_words = (int64_t)p2p_mailbox_words(copy_words, m, false);
    P->mbox_bytes = sizeof(unsigned long long) * (size_t)P->rvp * (size_t)P->p2p_vrow_words;
    CUDA_TRY(cudaMalloc(&P->mbox_alloc, P->mbox_bytes));
    CUDA_TRY(cudaMemsetAsync(P->mbox_alloc, 0, P->mbox_bytes, s));
    TRY(alloc_err(P));
    CUDA_TRY(cudaMalloc(&P->d_epoch, sizeof(unsigned int) * P->p2p_nslices * P->rvp));
    CUDA_TRY(cudaMemsetAsync(P->d_epoch, 0, sizeof(unsigned int) * P->p2p_nslices * P->rvp, s));
    P->p2p = true;
  }
  if (flags & CTRI_FLAG_TIMING) {
    P->ev.resize(EV_COUNT);
    for (auto& e : P->ev) CUDA_TRY(cudaEventCreate(&e));
  }
  // local solve; + window pass (one partition column-serial); + reduced kernel and window pass
  // (nparts > 1, or the vp partitions of one GPU); the on-chip single partition is complete
  P->launches_per_solve = 1 + (p > 1 || P->vp > 1 ? 2 : (P->local_kernel == 4 ? 0 : 1));
  CUDA_TRY(cudaStreamSynchronize(s));
  return CTRI_OK;
}

// Map every peer's mailbox: CUDA IPC handles all-gathered over the plan's NCCL communicator.
// The all-gather is issued after this rank zeroed its mailbox (same stream), so when it
// completes every rank's flags are initialised.
ctri_status p2p_connect_ipc(Plan* P, cudaStream_t s) {
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, P->mbox_alloc));
  char* d_h = nullptr;
  CUDA_TRY(cudaMalloc(&d_h, sizeof(h) * P->p));
  std::vector<char> all(sizeof(h) * P->p);
  ctri_status st = CTRI_OK;
  do {
    if (cudaMemcpyAsync(d_h + sizeof(h) * P->rank, &h, sizeof(h), cudaMemcpyHostToDevice, s) != cudaSuccess) { st = fail(CTRI_ERR_CUDA, "ipc handle upload"); break; }
    if (ncclAllGather(d_h + sizeof(h) * P->rank, d_h, sizeof(h), ncclChar, P->comm, s) != ncclSuccess) { st = fail(CTRI_ERR_NCCL, "ipc handle all-gather"); break; }
    if (cudaMemcpyAsync(all.data(), d_h, all.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) { st = fail(CTRI_ERR_CUDA, "ipc handle download"); break; }
  } while (0);
  cudaFree(d_h);
  if (st != CTRI_OK) return st;
  P->peer_alloc.assign(P->p, nullptr);
  P->peer_ipc.assign(P->p, false);
  for (int r = 0; r < P->p; ++r) {
    if (r == P->rank) { P->peer_alloc[r] = P->mbox_alloc; continue; }
    cudaIpcMemHandle_t hr;
    std::memcpy(&hr, all.data() + sizeof(h) * r, sizeof(h));
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, hr, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    P->peer_alloc[r] = ptr;
    P->peer_ipc[r] = true;
  }
  return CTRI_OK;
}

void p2p_args(const Plan& P0, P2PArgs* A) {
  std::memset(A, 0, sizeof(*A));
  A->p = P0.p * P0.rvp;  // reduced rows: nparts x virtual rows
  A->q = (int)P0.sched.steps.size();
  A->allgather = P0.allgather ? 1 : 0;
  A->pdl = (!P0.loopback && !knob_no_pdl()) ? 1 : 0;
  A->copy_words = p2p_copy_words(P0.lay.m(), A->q, A->p, P0.allgather || P0.r == 2, P0.r == 2 ? 4 : 2);
  if (P0.r == 2) {
    A->copy_words = P0.p2p_copy;
    A->q = P0.ppcr ? P0.ppcr_steps : 0;
  }
  A->cyclic = P0.cyclic;
  A->nslices = P0.p2p_nslices;
  A->m = P0.lay.m();
  A->slice_cols = (A->m + A->nslices - 1) / A->nslices;
  A->full = ((P0.flags & CTRI_FLAG_FULL_BACKSUB) || (2 * P0.window >= P0.lay.n / P0.rvp - 1)) ? 1 : 0;
  A->W = P0.window;
  A->lay = P0.lay;
  A->l = P0.bands.l;
  A->u = P0.bands.u;
  A->S = P0.d_S;
  A->R = P0.d_R;
  A->err = P0.d_err;
  A->deadline_ns = P0.deadline_ns;
  A->test_drop_rank = P0.test_drop_rank;
}

// Row `v` of this rank's virtual partitions (v = 0 without them): global reduced row
// rank * vp + v, its slab at row v * n_v (outer == 1 whenever vp > 1 with nparts > 1), its
// plane segment, mailbox and epochs.
void p2p_fill_rank(const Plan& P, double* x, P2PRank* R, int v = 0) {
  const int vp = P.rvp, pr = P.p * vp;
  const int64_t m = P.lay.m();
  const int g = P.rank * vp + v;
  R->rank = g;
  R->x = x ? x + (int64_t)v * (P.lay.n / vp) * P.lay.inner : nullptr;
  R->yf = P.yf + (int64_t)v * m;
  R->yl = P.yl + (int64_t)v * m;
  R->bt = P.bt + (int64_t)v * m;
  R->xnext = P.r == 2 ? P.d_xnext2 + (int64_t)v * 2 * m : P.xt_next + (int64_t)v * m;
  R->planes4 = P.d_planes4 ? P.d_planes4 + (int64_t)v * m : nullptr;  // [4][pstride], row v's segment
  R->pstride = (P.r == 2 && P.p > 1) ? m * vp : m;
  R->ainv = P.d_ainv;
  R->mbox = reinterpret_cast<unsigned long long*>(P.mbox_alloc) + P.p2p_off + (int64_t)v * P.p2p_vrow_words;
  R->epoch = P.d_epoch + (int64_t)v * P.p2p_nslices;
  R->f = nullptr;
  R->halo_lo = P.halo_lo;
  R->halo_hi = P.halo_hi;
  for (int r = 0; r < kMaxP2PRanks; ++r) R->peer_mbox[r] = nullptr;
  for (int r = 0; r < pr; ++r)
    R->peer_mbox[r] = reinterpret_cast<unsigned long long*>(P.peer_alloc[r / vp]) + P.p2p_off +
                      (int64_t)(r % vp) * P.p2p_vrow_words;
  for (int r = 0; r < kMaxAG; ++r) {
    R->ag0[r] = R->ag1[r] = 0.0;
    if (!P.allgather || r >= P.p) continue;
    const int nx = P.rank + 1;  // x~_{i+1}: rank i+1, wrapping to 0 (cyclic) or absent (acyclic)
    R->ag0[r] = P.ainv[(size_t)P.rank * P.p + r];
    if (nx < P.p || P.cyclic) R->ag1[r] = P.ainv[(size_t)(nx % P.p) * P.p + r];
  }
  R->ppcr = P.d_ppcr ? P.d_ppcr + (size_t)v * 12 * P.ppcr_steps : nullptr;
  if (P.r == 2) {
    for (int s = 0; s < kMaxP2PSteps; ++s) {
      const size_t k = (size_t)v * kMaxP2PSteps + s;
      R->step[s] = k < P.pstep.size() ? P.pstep[k] : P2PStep{1.0, 0.0, 0.0, -1, -1, -1, -1, 0, 0};
    }
    return;
  }
  const Schedule& sc = P.sched;
  for (int s = 0; s < kMaxP2PSteps; ++s) {
    P2PStep& t = R->step[s];
    t = P2PStep{1.0, 0.0, 0.0, -1, -1, -1, -1, 0, 0};
    if (s >= (int)sc.steps.size()) continue;
    const SchedEntry& e = sc.steps[s][g];
    t.w = e.w;
    t.c0 = e.c[0];
    t.c1 = e.c[1];
    t.src0 = (int8_t)e.src[0];
    t.src1 = (int8_t)e.src[1];
    int nd = 0;  // rows that read this row's value in step s, and their slot
    for (int i = 0; i < pr; ++i)
      for (int k = 0; k < 2; ++k)
        if (sc.steps[s][i].src[k] == g) {
          if (nd == 0) { t.dst0 = (int8_t)i; t.dslot0 = (int8_t)k; }
          else { t.dst1 = (int8_t)i; t.dslot1 = (int8_t)k; }
          ++nd;
        }
  }
}

// messages this rank sends per solve, and dependent exchange rounds, from the schedule
void schedule_counts(const Plan& P, int* sends, int* rounds) {
  if (P.r == 2 && P.ppcr) {  // y, block-PCR steps (2 planes per message), x
    int sd = (has_right(P) ? 2 : 0) + (has_left(P) ? 2 : 0), rd = 2;
    for (int k = 0; k < P.ppcr_steps; ++k) {
      const P2PStep& t = P.pstep[k];
      sd += 2 * ((t.dst0 >= 0 ? 1 : 0) + (t.dst1 >= 0 ? 1 : 0));
      if (t.src0 >= 0 || t.src1 >= 0 || t.dst0 >= 0 || t.dst1 >= 0) ++rd;  // (the fold is local)
    }
    *sends = sd;
    *rounds = rd;
    return;
  }
  if (P.allgather || P.r == 2) {  // one round: 2 (4 for r = 2) planes to each of the p - 1 peers
    *sends = 2 * P.r * (P.p - 1);
    *rounds = 1;
    return;
  }
  // messages leaving this GPU (its vp virtual rows to rows of other ranks), dependent rounds
  const Schedule& sc = P.sched;
  const int vp = P.rvp, pr = P.p * vp;
  auto owner = [&](int row) { return row / vp; };
  int sd = 0, rd = 2;
  for (int v = 0; v < vp; ++v) {
    const int g = P.rank * vp + v;
    const int rt = P.cyclic ? (g + 1) % pr : (g + 1 < pr ? g + 1 : -1);
    const int lt = P.cyclic ? (g + pr - 1) % pr : (g > 0 ? g - 1 : -1);
    if (rt >= 0 && owner(rt) != P.rank) ++sd;  // y round
    if (lt >= 0 && owner(lt) != P.rank) ++sd;  // x~ round
  }
  for (size_t s = 0; s < sc.steps.size(); ++s) {
    bool any = false;
    for (int i = 0; i < pr; ++i)
      for (int k = 0; k < 2; ++k) {
        const int src = sc.steps[s][i].src[k];
        if (src >= 0) any = true;
        if (src >= 0 && owner(src) == P.rank && owner(i) != P.rank) ++sd;
      }
    rd += any ? 1 : 0;
  }
  *sends = sd;
  *rounds = rd;
}

// ---------------- exchanges ----------------
struct Xfer {
  int send_to;        // -1: none
  const double* sbuf;
  int recv_from;      // -1: none
  double* rbuf;
  int64_t count;
};

// NCCL: one group per round (all of this rank's sends and receives of the round).
ctri_status exchange_nccl(Plan& P, const std::vector<Xfer>& xs, cudaStream_t s) {
  NCCL_TRY(ncclGroupStart());
  for (const Xfer& x : xs) {
    if (x.send_to >= 0) NCCL_TRY(ncclSend(x.sbuf, (size_t)x.count, ncclDouble, x.send_to, P.comm, s));
    if (x.recv_from >= 0)
      NCCL_TRY(ncclRecv(x.rbuf, (size_t)x.count, ncclDouble, x.recv_from, P.comm, s));
  }
  NCCL_TRY(ncclGroupEnd());
  return CTRI_OK;
}

// Per-rank transfer lists of each round (shared by NCCL and loopback).
std::vector<Xfer> round_y(Plan& P) {  // y_{i-1}[last]: i -> i+1
  Xfer x{has_right(P) ? wrap(P, P.rank + 1) : -1, P.yl, has_left(P) ? wrap(P, P.rank - 1) : -1,
         P.yl_prev, P.lay.m()};
  return {x};
}
std::vector<Xfer> round_stage(Plan& P, int k) {  // b^ with partners i -+ 2^k
  const int s = 1 << k;
  const int64_t m = P.lay.m();
  int lm = P.rank - s, lp = P.rank + s;
  if (P.cyclic) {
    lm = wrap(P, lm);
    lp = wrap(P, lp);
  } else {
    if (lm < 0) lm = -1;
    if (lp >= P.p) lp = -1;
  }
  if (lm >= 0 && lm == lp) return {Xfer{lp, P.bh, lm, P.recv_m, m}};  // s = p/2: single partner
  std::vector<Xfer> v;
  // order: send to i+s / recv from i-s, then send to i-s / recv from i+s
  v.push_back(Xfer{lp, P.bh, lm, P.recv_m, m});
  v.push_back(Xfer{lm, P.bh, lp, P.recv_p, m});
  return v;
}
std::vector<Xfer> round_x(Plan& P) {  // x~_{i+1}: i+1 -> i
  Xfer x{has_left(P) ? wrap(P, P.rank - 1) : -1, P.xt, has_right(P) ? wrap(P, P.rank + 1) : -1,
         P.xt_next, P.lay.m()};
  return {x};
}
std::vector<Xfer> round_halo(Plan& P) {
  const int64_t m2 = 2 * P.lay.m();
  return {Xfer{wrap(P, P.rank - 1), P.send_lo, wrap(P, P.rank + 1), P.halo_hi, m2},
          Xfer{wrap(P, P.rank + 1), P.send_hi, wrap(P, P.rank - 1), P.halo_lo, m2}};
}

// Loopback: for each rank r and each of its receives, copy from the sender's buffer.  The
// sender's buffer is identified by matching the sender's own transfer list.
template <typename RoundFn>
ctri_status exchange_loopback(std::vector<Plan*>& G, RoundFn fn, cudaStream_t s) {
  const int p = (int)G.size();
  std::vector<std::vector<Xfer>> lists(p);
  for (int r = 0; r < p; ++r) lists[r] = fn(*G[r]);
  for (int r = 0; r < p; ++r) {
    // receives of rank r are matched in order with sends of the peer addressed to r
    std::vector<int> used(p, 0);
    for (const Xfer& x : lists[r]) {
      if (x.recv_from < 0) continue;
      const int q = x.recv_from;
      int seen = 0;
      const double* src = nullptr;
      for (const Xfer& y : lists[q]) {
        if (y.send_to == r) {
          if (seen == used[q]) { src = y.sbuf; break; }
          ++seen;
        }
      }
      if (!src) return fail(CTRI_ERR_INVALID_ARG, "loopback: unmatched receive");
      ++used[q];
      CUDA_TRY(cudaMemcpyAsync(x.rbuf, src, x.count * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  }
  return CTRI_OK;
}

void record(Plan& P, int slot, cudaStream_t s) {
  if (P.ev.empty()) return;
  // inside a CUDA-graph capture the phase events become external event-record nodes, so
  // ctri_get_stats can still read them after a replay
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(P.ev[slot], s, cudaEventRecordExternal);
  else
    cudaEventRecord(P.ev[slot], s);
}

// (a1) local solve; with `deriv` the tile kernel reads f and forms the stencil RHS itself (a0).
ctri_status local_phase(Plan& P, const double* b, double* x, cudaStream_t s,
                        const Stencil5* st = nullptr) {
  cudaError_t e = (P.local_kernel >= 1) ? launch_tile(P, b, x, s, st)
                                        : launch_local_generic(P, b, x, s);
  if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("local solve launch: ") + cudaGetErrorString(e));
  return CTRI_OK;
}

ctri_status stage_kernel(Plan& P, int k, cudaStream_t s) {
  const bool last = (k == P.gpcr.stages - 1);
  // single-partner stage: both couplings read recv_m
  double* saved = P.recv_p;
  std::vector<Xfer> r = round_stage(P, k);
  if (r.size() == 1) P.recv_p = P.recv_m;
  cudaError_t e = launch_pcr_stage(P, k, last, s);
  P.recv_p = saved;
  if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("pcr stage: ") + cudaGetErrorString(e));
  return CTRI_OK;
}

ctri_status penta_solve_group(std::vector<Plan*>& G, const double* const* b, double* const* x,
                              cudaStream_t s);

// The whole solve for a set of co-scheduled plans: one plan (NCCL) or a loopback group.
ctri_status solve_group(std::vector<Plan*>& G, const double* const* b, double* const* x,
                        cudaStream_t s, const Stencil5* st = nullptr) {
  if (G[0]->r == 2) {
    if (st) return fail(CTRI_ERR_UNSUPPORTED, "pentadiagonal plans have no derivative path");
    return penta_solve_group(G, b, x, s);
  }
  const bool nccl = !G[0]->loopback;
  Plan& P0 = *G[0];
  TRY(check_poisoned(G));
  for (size_t r = 0; r < G.size(); ++r) {
    if (!b[r] || !x[r]) return fail(CTRI_ERR_INVALID_ARG, "NULL b or x");
    if (((uintptr_t)b[r] | (uintptr_t)x[r]) & 15)
      return fail(CTRI_ERR_INVALID_ARG, "b and x must be 16-byte aligned");
  }
  for (Plan* P : G) P->solves++;
  record(P0, EV_START, s);
  for (size_t r = 0; r < G.size(); ++r) TRY(local_phase(*G[r], b[r], x[r], s, st));
  record(P0, EV_LOCAL, s);
  if (P0.fused && !st) {  // (a2)-(a4) ran inside the tile kernel
    record(P0, EV_BACK, s);
    for (Plan* P : G) P->timed_valid = !P->ev.empty();
    return CTRI_OK;
  }
  if (P0.p == 1) {
    if (P0.vp > 1 && !P0.vchain) {  // (a2)-(a4) across the virtual partitions of this slab
      for (size_t r = 0; r < G.size(); ++r) {
        cudaError_t e = launch_reduced_local(*G[r], x[r], s);
        if (e == cudaSuccess) e = launch_window(*G[r], x[r], nullptr, s);
        if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("local reduced: ") + cudaGetErrorString(e));
      }
      record(P0, EV_BACK, s);
      for (Plan* P : G) P->timed_valid = !P->ev.empty();
    }
    return CTRI_OK;
  }
  if (P0.p2p) {  // fused device-initiated (a2)-(a4)
    P2PArgs A;
    p2p_args(P0, &A);
    const int nrows = (int)G.size() * P0.rvp;  // rows launched together (ranks x virtual rows)
    const int grid = A.nslices * nrows;
    const bool env_trace = knob_p2p_trace();
    if ((env_trace || !P0.ev.empty()) && !P0.d_trace) {  // per-round stamps (CTRI_FLAG_TIMING)
      CUDA_TRY(cudaMalloc(&P0.d_trace, sizeof(unsigned long long) * kP2PTrace * grid));
      CUDA_TRY(cudaMemsetAsync(P0.d_trace, 0, sizeof(unsigned long long) * kP2PTrace * grid, s));
      P0.trace_ctas = grid;
    }
    A.trace = P0.d_trace;
    for (size_t r = 0; r < G.size(); ++r)
      for (int v = 0; v < P0.rvp; ++v) p2p_fill_rank(*G[r], x[r], &A.rk[r * P0.rvp + v], v);
    // CTAs of different reduced rows on this GPU wait on each other (loopback ranks, virtual
    // rows): one cooperative grid guarantees they are co-resident even when other work shares
    // the GPU.  A single row per GPU waits only on peers and is launched with PDL instead.
    cudaError_t e = launch_reduced_p2p(A, nrows, s, nrows);
    if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("p2p reduced kernel: ") + cudaGetErrorString(e));
    record(P0, EV_XX, s);
    for (size_t r = 0; r < G.size(); ++r) {  // (a4) window pass of every rank (all its slabs)
      e = launch_window(*G[r], x[r], G[r]->xt_next + (int64_t)(G[r]->rvp - 1) * G[r]->lay.m(), s);
      if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("window: ") + cudaGetErrorString(e));
    }
    if (P0.d_trace && env_trace) {  // measurement only: per-phase spread across CTAs on stderr
      std::vector<unsigned long long> t((size_t)kP2PTrace * grid);
      CUDA_TRY(cudaMemcpyAsync(t.data(), P0.d_trace, t.size() * 8, cudaMemcpyDeviceToHost, s));
      CUDA_TRY(cudaStreamSynchronize(s));
      unsigned long long t0 = ~0ull;
      for (int b = 0; b < grid; ++b) t0 = std::min(t0, t[(size_t)kP2PTrace * b]);
      std::fprintf(stderr, "[p2p trace rank %d solve %llu]", P0.rank, (unsigned long long)P0.solves);
      const int slots[5] = {kTrStart, kTrYSent, kTrYRecv, kTrXRecv, kTrEnd};
      const char* nm[5] = {"start", "y_sent", "y_recv", "x_recv", "end"};
      for (int k = 0; k < 5; ++k) {
        std::vector<double> v;
        for (int b = 0; b < grid; ++b) v.push_back((t[(size_t)kP2PTrace * b + slots[k]] - t0) * 1e-3);
        std::sort(v.begin(), v.end());
        std::fprintf(stderr, " %s %.1f/%.1f/%.1f", nm[k], v.front(), v[v.size() / 2], v.back());
      }
      std::fprintf(stderr, " us\n");
    }
    record(P0, EV_BACK, s);
    for (Plan* P : G) P->timed_valid = !P->ev.empty();
    return CTRI_OK;
  }
  // (a2) neighbour exchange of y_{i-1}[last] and b^ assembly
  if (nccl) TRY(exchange_nccl(P0, round_y(P0), s));
  else TRY(exchange_loopback(G, [](Plan& P) { return round_y(P); }, s));
  record(P0, EV_YX, s);
  for (Plan* P : G) {
    cudaError_t e = launch_bhat(*P, s);
    if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, cudaGetErrorString(e));
  }
  record(P0, EV_BHAT, s);
  // (a3) distributed PCR stages
  for (int k = 0; k < P0.gpcr.stages; ++k) {
    if (nccl) TRY(exchange_nccl(P0, round_stage(P0, k), s));
    else TRY(exchange_loopback(G, [k](Plan& P) { return round_stage(P, k); }, s));
    for (Plan* P : G) TRY(stage_kernel(*P, k, s));
    record(P0, EV_STAGE0 + k, s);
  }
  // (a4) x~_{i+1} exchange and back-substitution
  if (nccl) TRY(exchange_nccl(P0, round_x(P0), s));
  else TRY(exchange_loopback(G, [](Plan& P) { return round_x(P); }, s));
  record(P0, EV_XX, s);
  for (size_t r = 0; r < G.size(); ++r) {
    cudaError_t e = launch_backsub(*G[r], x[r], s);
    if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, cudaGetErrorString(e));
  }
  record(P0, EV_BACK, s);
  for (Plan* P : G) P->timed_valid = !P->ev.empty();
  return CTRI_OK;
}

// A compact scheme: df = A^{-1} (five-point periodic stencil of f); halos from the neighbours.
// Pentadiagonal solve of a plan group (one plan, or a loopback group).
ctri_status penta_solve_group(std::vector<Plan*>& G, const double* const* b, double* const* x,
                              cudaStream_t s) {
  Plan& P0 = *G[0];
  TRY(check_poisoned(G));
  for (size_t r = 0; r < G.size(); ++r) {
    if (!b[r] || !x[r]) return fail(CTRI_ERR_INVALID_ARG, "NULL b or x");
    if (((uintptr_t)b[r] | (uintptr_t)x[r]) & 15)  // TMA tiles, 16-byte window pairs
      return fail(CTRI_ERR_INVALID_ARG, "b and x must be 16-byte aligned");
  }
  for (Plan* P : G) P->solves++;
  record(P0, EV_START, s);
  for (size_t r = 0; r < G.size(); ++r) {
    cudaError_t e = G[r]->local_kernel == 4 ? launch_ptile(*G[r], b[r], x[r], s)
                                            : launch_penta_local(*G[r], b[r], x[r], s);
    if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("penta local: ") + cudaGetErrorString(e));
  }
  record(P0, EV_LOCAL, s);
  if (P0.p == 1 && P0.local_kernel == 4 && P0.vp == 1) {  // one partition solved completely on chip
    record(P0, EV_BACK, s);
    for (Plan* P : G) P->timed_valid = !P->ev.empty();
    return CTRI_OK;
  }
  if (P0.p == 1 && P0.vp > 1) {  // (a2)+(a3) over this GPU's partitions: x~ into rows 0, 1 of each
    for (size_t r = 0; r < G.size(); ++r) {
      cudaError_t e = launch_penta_reduced_local(*G[r], x[r], s);
      if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("penta reduced: ") + cudaGetErrorString(e));
    }
    record(P0, EV_XX, s);
  }
  if (P0.p > 1) {
    P2PArgs A;
    p2p_args(P0, &A);
    const int nrows = (int)G.size() * P0.rvp;  // block rows launched together (ranks x virtual rows)
    const int grid = A.nslices * nrows;
    if (!P0.ev.empty() && !P0.d_trace) {  // per-round stamps (CTRI_FLAG_TIMING)
      CUDA_TRY(cudaMalloc(&P0.d_trace, sizeof(unsigned long long) * kP2PTrace * grid));
      CUDA_TRY(cudaMemsetAsync(P0.d_trace, 0, sizeof(unsigned long long) * kP2PTrace * grid, s));
      P0.trace_ctas = grid;
    }
    A.trace = P0.d_trace;
    for (size_t r = 0; r < G.size(); ++r)
      for (int v = 0; v < P0.rvp; ++v) p2p_fill_rank(*G[r], x[r], &A.rk[r * P0.rvp + v], v);
    cudaError_t e = P0.ppcr ? launch_reduced_penta_pcr(A, nrows, s)
                            : launch_reduced_allgather_r2(A, (int)G.size(), s);
    if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("penta reduced: ") + cudaGetErrorString(e));
    record(P0, EV_XX, s);
  }
  for (size_t r = 0; r < G.size(); ++r) {
    cudaError_t e = launch_penta_window(*G[r], x[r], s);
    if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("penta window: ") + cudaGetErrorString(e));
  }
  record(P0, EV_BACK, s);
  for (Plan* P : G) P->timed_valid = !P->ev.empty();
  return CTRI_OK;
}

ctri_status deriv_group(std::vector<Plan*>& G, const double* const* f, double* const* df,
                        const double coef[5], cudaStream_t s) {
  if (G[0]->r == 2) return fail(CTRI_ERR_UNSUPPORTED, "pentadiagonal plans have no derivative path");
  for (size_t r = 0; r < G.size(); ++r) {
    Plan& P = *G[r];
    if (!(P.flags & CTRI_FLAG_DERIV)) return fail(CTRI_ERR_INVALID_ARG, "plan lacks CTRI_FLAG_DERIV");
    if (!f[r] || !df[r] || f[r] == df[r]) return fail(CTRI_ERR_INVALID_ARG, "f/df NULL or aliased");
  }
  if (!coef) return fail(CTRI_ERR_INVALID_ARG, "NULL coef");
  for (int k = 0; k < 5; ++k)
    if (!std::isfinite(coef[k])) return fail(CTRI_ERR_INVALID_ARG, "non-finite stencil coefficient");
  const Stencil5 st = make_stencil5(coef);
  bool fused = true;
  for (Plan* P : G) fused = fused && P->local_kernel == 1 && P->tile.deriv_ok;
  // halo planes for the host-issued exchange (with one partition the fused kernel loads the
  // slab's own wrap rows by TMA, and the unfused stencil wraps by itself)
  const bool need_pack = G[0]->p > 1 && !G[0]->p2p;
  if (need_pack) {
    for (size_t r = 0; r < G.size(); ++r) {
      cudaError_t e = launch_pack_halo(*G[r], f[r], s);
      if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, cudaGetErrorString(e));
    }
  }
  TRY(check_poisoned(G));
  if (G[0]->p > 1 && G[0]->p2p) {  // halo rows as LL words over the P2P mailboxes
    P2PArgs A;
    p2p_args(*G[0], &A);
    A.p = G[0]->p;  // real ranks (not virtual rows): slab neighbours
    for (size_t r = 0; r < G.size(); ++r) {
      const Plan& P = *G[r];
      p2p_fill_rank(P, nullptr, &A.rk[r]);
      A.rk[r].rank = P.rank;
      A.rk[r].f = f[r];
      A.rk[r].epoch = P.d_hepoch;
      A.rk[r].mbox = reinterpret_cast<unsigned long long*>(P.mbox_alloc) + P.halo_off;
      for (int j = 0; j < kMaxP2PRanks; ++j)
        A.rk[r].peer_mbox[j] = j < P.p ? reinterpret_cast<unsigned long long*>(P.peer_alloc[j]) + P.halo_off : nullptr;
    }
    cudaError_t e = launch_halo_p2p(A, (int)G.size(), s);
    if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, std::string("p2p halo: ") + cudaGetErrorString(e));
  } else if (G[0]->p > 1) {
    if (!G[0]->loopback) TRY(exchange_nccl(*G[0], round_halo(*G[0]), s));
    else TRY(exchange_loopback(G, [](Plan& P) { return round_halo(P); }, s));
  }
  if (fused)  // (a0) fused into (a1): f read once, df written once
    return solve_group(G, f, df, s, &st);
  for (size_t r = 0; r < G.size(); ++r) {
    cudaError_t e = launch_stencil(*G[r], f[r], df[r], st, s);
    if (e != cudaSuccess) return fail(CTRI_ERR_CUDA, cudaGetErrorString(e));
  }
  return solve_group(G, df, df, s);
}

float elapsed(const Plan& P, int a, int b) {
  float ms = -1.f;
  if (cudaEventElapsedTime(&ms, P.ev[a], P.ev[b]) != cudaSuccess) {
    cudaGetLastError();
    return -1.f;
  }
  return ms * 1000.f;
}
}  // namespace

// ====================================== ABI =============================================
extern "C" {

const char* ctri_status_string(ctri_status s) {
  switch (s) {
    case CTRI_OK: return "CTRI_OK";
    case CTRI_ERR_INVALID_ARG: return "CTRI_ERR_INVALID_ARG";
    case CTRI_ERR_UNSUPPORTED: return "CTRI_ERR_UNSUPPORTED";
    case CTRI_ERR_SINGULAR: return "CTRI_ERR_SINGULAR";
    case CTRI_ERR_PARTITION_TOO_SMALL: return "CTRI_ERR_PARTITION_TOO_SMALL";
    case CTRI_ERR_CUDA: return "CTRI_ERR_CUDA";
    case CTRI_ERR_NCCL: return "CTRI_ERR_NCCL";
    case CTRI_ERR_OOM: return "CTRI_ERR_OOM";
  }
  return "CTRI_ERR_UNKNOWN";
}

const char* ctri_last_error(void) { return g_err.c_str(); }

int ctri_abi_version(void) { return CTRI_ABI_VERSION; }

ctri_status ctri_get_unique_id(void* out128) {
  if (!out128) return fail(CTRI_ERR_INVALID_ARG, "NULL out");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
  return CTRI_OK;
}

ctri_status ctri_plan_create(ctri_plan* out, const int64_t global_dims[3], int solve_dim,
                             int nparts, int rank, const double bands[3], int cyclic,
                             const void* nccl_unique_id, uint32_t flags, ctri_stream stream) {
  if (!out) return fail(CTRI_ERR_INVALID_ARG, "NULL out");
  *out = nullptr;
  if (nparts > 1 && !nccl_unique_id)
    return fail(CTRI_ERR_INVALID_ARG, "nparts > 1 needs an NCCL unique id");
  std::unique_ptr<Plan, void (*)(Plan*)> P(new Plan(), free_plan);
  ctri_status st = plan_init(P.get(), global_dims, solve_dim, nparts, rank, bands, cyclic, flags,
                             (cudaStream_t)stream);
  if (st != CTRI_OK) return st;
  if (nparts > 1) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    NCCL_TRY(ncclCommInitRank(&P->comm, nparts, id, rank));
    if (P->p2p) {
      ctri_status cs = p2p_connect_ipc(P.get(), (cudaStream_t)stream);
      if (cs != CTRI_OK) return cs;
    }
  }
  *out = reinterpret_cast<ctri_plan>(P.release());
  return CTRI_OK;
}

ctri_status ctri_plan_create_loopback(ctri_plan* plans, int nparts, const int64_t global_dims[3],
                                      int solve_dim, const double bands[3], int cyclic,
                                      uint32_t flags, ctri_stream stream) {
  if (!plans || nparts < 1) return fail(CTRI_ERR_INVALID_ARG, "bad plans/nparts");
  std::vector<Plan*> made;
  for (int r = 0; r < nparts; ++r) {
    Plan* P = new Plan();
    P->loopback = true;
    ctri_status st = plan_init(P, global_dims, solve_dim, nparts, r, bands, cyclic, flags,
                               (cudaStream_t)stream);
    if (st != CTRI_OK) {
      free_plan(P);
      for (Plan* q : made) free_plan(q);
      return st;
    }
    made.push_back(P);
  }
  for (int r = 0; r < nparts; ++r) {
    made[r]->group = made;
    if (made[r]->p2p) {
      made[r]->peer_alloc.assign(nparts, nullptr);
      made[r]->peer_ipc.assign(nparts, false);
      for (int q = 0; q < nparts; ++q) made[r]->peer_alloc[q] = made[q]->mbox_alloc;
    }
    plans[r] = reinterpret_cast<ctri_plan>(made[r]);
  }
  return CTRI_OK;
}

ctri_status ctri_plan_create_penta(ctri_plan* out, const int64_t global_dims[3], int solve_dim,
                                   int nparts, int rank, const double bands[5], int cyclic,
                                   const void* nccl_unique_id, uint32_t flags, ctri_stream stream) {
  if (!out) return fail(CTRI_ERR_INVALID_ARG, "NULL out");
  *out = nullptr;
  if (nparts > 1 && !nccl_unique_id)
    return fail(CTRI_ERR_INVALID_ARG, "nparts > 1 needs an NCCL unique id");
  std::unique_ptr<Plan, void (*)(Plan*)> P(new Plan(), free_plan);
  ctri_status st = penta_init(P.get(), global_dims, solve_dim, nparts, rank, bands, cyclic, flags,
                              (cudaStream_t)stream);
  if (st != CTRI_OK) return st;
  if (nparts > 1) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    NCCL_TRY(ncclCommInitRank(&P->comm, nparts, id, rank));
    ctri_status cs = p2p_connect_ipc(P.get(), (cudaStream_t)stream);
    if (cs != CTRI_OK) return cs;
  }
  *out = reinterpret_cast<ctri_plan>(P.release());
  return CTRI_OK;
}

ctri_status ctri_plan_create_penta_loopback(ctri_plan* plans, int nparts,
                                            const int64_t global_dims[3], int solve_dim,
                                            const double bands[5], int cyclic, uint32_t flags,
                                            ctri_stream stream) {
  if (!plans || nparts < 1) return fail(CTRI_ERR_INVALID_ARG, "bad plans/nparts");
  std::vector<Plan*> made;
  for (int r = 0; r < nparts; ++r) {
    Plan* P = new Plan();
    P->loopback = true;
    ctri_status st = penta_init(P, global_dims, solve_dim, nparts, r, bands, cyclic, flags,
                                (cudaStream_t)stream);
    if (st != CTRI_OK) {
      free_plan(P);
      for (Plan* q : made) free_plan(q);
      return st;
    }
    made.push_back(P);
  }
  for (int r = 0; r < nparts; ++r) {
    made[r]->group = made;
    if (made[r]->p2p) {
      made[r]->peer_alloc.assign(nparts, nullptr);
      made[r]->peer_ipc.assign(nparts, false);
      for (int q = 0; q < nparts; ++q) made[r]->peer_alloc[q] = made[q]->mbox_alloc;
    }
    plans[r] = reinterpret_cast<ctri_plan>(made[r]);
  }
  return CTRI_OK;
}

ctri_status ctri_solve(ctri_plan plan, const double* b, double* x, ctri_stream stream) {
  if (!plan) return fail(CTRI_ERR_INVALID_ARG, "NULL plan");
  Plan* P = reinterpret_cast<Plan*>(plan);
  if (P->loopback && P->p > 1) return fail(CTRI_ERR_INVALID_ARG, "loopback plan: use ctri_solve_loopback");
  std::vector<Plan*> G{P};
  return solve_group(G, &b, &x, (cudaStream_t)stream);
}

ctri_status ctri_solve_loopback(const ctri_plan* plans, int nparts, const double* const* b,
                                double* const* x, ctri_stream stream) {
  if (!plans || !b || !x || nparts < 1) return fail(CTRI_ERR_INVALID_ARG, "NULL arguments");
  std::vector<Plan*> G(nparts);
  for (int r = 0; r < nparts; ++r) {
    G[r] = reinterpret_cast<Plan*>(plans[r]);
    if (!G[r] || G[r]->rank != r || G[r]->p != nparts || !G[r]->loopback)
      return fail(CTRI_ERR_INVALID_ARG, "plans must be one loopback group in rank order");
  }
  return solve_group(G, b, x, (cudaStream_t)stream);
}

// Choose the e2e pipeline for a one-partition plan: column chunks that are independent
// problems of the same method (a sub-plan of the chunk's shape solves each).
static ctri_status e2e_setup(Plan* P, cudaStream_t s) {
  P->e2e_mode = 0;
  const int64_t outer = P->lay.outer, n = P->lay.n, inner = P->lay.inner;
  const size_t bytes = (size_t)P->lay.elems() * sizeof(double);
  int nch = 16;  // measured on B200 (cfg2, pinned host): 4 -> 110 ms, 8 -> 101, 16 -> 94, 32 -> 92
  if (const char* e = std::getenv("CTRI_E2E_CHUNKS")) nch = std::atoi(e);  // measurement knob
  if (P->p != 1 || P->loopback || nch < 2 || bytes < ((size_t)256 << 20)) return CTRI_OK;
  int64_t dims[3];
  int mode = 0;
  if (outer % nch == 0) {
    mode = 1;
    dims[0] = outer / nch, dims[1] = n, dims[2] = inner;
  } else if (outer == 1 && inner % nch == 0 && (inner / nch) % 2 == 0) {
    mode = 2;
    dims[0] = 1, dims[1] = n, dims[2] = inner / nch;
  } else {
    return CTRI_OK;
  }
  Plan* S = new Plan();
  const uint32_t fl = P->flags & (CTRI_FLAG_FULL_BACKSUB | CTRI_FLAG_GENERIC_LOCAL);
  ctri_status st;
  if (P->r == 2) {
    st = penta_init(S, dims, 1, 1, 0, P->bands5, P->cyclic, fl, s);
  } else {
    const double bd[3] = {P->bands.l, P->bands.d, P->bands.u};
    st = plan_init(S, dims, 1, 1, 0, bd, P->cyclic, fl, s);
  }
  if (st != CTRI_OK) {
    free_plan(S);
    g_err.clear();
    return CTRI_OK;  // no pipeline for this shape: sequential copies
  }
  P->e2e_sub = S;
  CUDA_TRY(cudaStreamCreateWithFlags(&P->e2e_h2d, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&P->e2e_d2h, cudaStreamNonBlocking));
  P->e2e_ev.resize(2 + 2 * (size_t)nch);
  for (auto& e : P->e2e_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  P->e2e_nch = nch;
  P->e2e_mode = mode;
  return CTRI_OK;
}

ctri_status ctri_solve_host(ctri_plan plan, const double* b_host, double* x_host,
                            ctri_stream stream) {
  if (!plan || !b_host || !x_host) return fail(CTRI_ERR_INVALID_ARG, "NULL argument");
  Plan* P = reinterpret_cast<Plan*>(plan);
  const size_t bytes = (size_t)P->lay.elems() * sizeof(double);
  if (!P->d_stage_b) {
    CUDA_TRY(cudaMalloc(&P->d_stage_b, bytes));
    CUDA_TRY(cudaMalloc(&P->d_stage_x, bytes));
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (P->e2e_mode < 0) TRY(e2e_setup(P, s));
  if (P->e2e_mode == 0) {
    CUDA_TRY(cudaMemcpyAsync(P->d_stage_b, b_host, bytes, cudaMemcpyHostToDevice, s));
    TRY(ctri_solve(plan, P->d_stage_b, P->d_stage_x, stream));
    CUDA_TRY(cudaMemcpyAsync(x_host, P->d_stage_x, bytes, cudaMemcpyDeviceToHost, s));
    return CTRI_OK;
  }
  // pipelined: H2D of chunk k+1 and D2H of chunk k-1 overlap the solve of chunk k
  const int nch = P->e2e_nch;
  const int64_t outer = P->lay.outer, n = P->lay.n, inner = P->lay.inner;
  const int64_t celems = P->lay.elems() / nch;  // elements per chunk (contiguous on the device)
  cudaEvent_t* ev = P->e2e_ev.data();
  cudaEvent_t *e_h2d = ev + 2, *e_sol = ev + 2 + nch;
  P->solves++;
  CUDA_TRY(cudaEventRecord(ev[0], s));
  CUDA_TRY(cudaStreamWaitEvent(P->e2e_h2d, ev[0], 0));
  CUDA_TRY(cudaStreamWaitEvent(P->e2e_d2h, ev[0], 0));
  const int64_t ic = inner / nch;
  for (int k = 0; k < nch; ++k) {
    double* db = P->d_stage_b + (size_t)k * celems;
    if (P->e2e_mode == 1) {
      CUDA_TRY(cudaMemcpyAsync(db, b_host + (size_t)k * celems, celems * sizeof(double),
                               cudaMemcpyHostToDevice, P->e2e_h2d));
    } else {  // columns [k*ic, (k+1)*ic) of every row (outer == 1)
      CUDA_TRY(cudaMemcpy2DAsync(db, ic * sizeof(double), b_host + (size_t)k * ic, inner * sizeof(double),
                                 ic * sizeof(double), n, cudaMemcpyHostToDevice, P->e2e_h2d));
    }
    CUDA_TRY(cudaEventRecord(e_h2d[k], P->e2e_h2d));
  }
  for (int k = 0; k < nch; ++k) {
    CUDA_TRY(cudaStreamWaitEvent(s, e_h2d[k], 0));
    std::vector<Plan*> G{P->e2e_sub};
    const double* bk = P->d_stage_b + (size_t)k * celems;
    double* xk = P->d_stage_x + (size_t)k * celems;
    TRY(solve_group(G, &bk, &xk, s));
    CUDA_TRY(cudaEventRecord(e_sol[k], s));
  }
  for (int k = 0; k < nch; ++k) {
    CUDA_TRY(cudaStreamWaitEvent(P->e2e_d2h, e_sol[k], 0));
    const double* dx = P->d_stage_x + (size_t)k * celems;
    if (P->e2e_mode == 1) {
      CUDA_TRY(cudaMemcpyAsync(x_host + (size_t)k * celems, dx, celems * sizeof(double),
                               cudaMemcpyDeviceToHost, P->e2e_d2h));
    } else {
      CUDA_TRY(cudaMemcpy2DAsync(x_host + (size_t)k * ic, inner * sizeof(double), dx, ic * sizeof(double),
                                 ic * sizeof(double), n, cudaMemcpyDeviceToHost, P->e2e_d2h));
    }
  }
  CUDA_TRY(cudaEventRecord(ev[1], P->e2e_d2h));
  CUDA_TRY(cudaStreamWaitEvent(s, ev[1], 0));
  (void)outer;
  return CTRI_OK;
}

// collocated compact first derivative as a five-point stencil
// a, bc NaN -> Lele's sixth-order pair (R8); h <= 0 or NaN -> 2 pi / N_global
static bool deriv_coef(const Plan& P, double a, double bc, double h, double c[5]) {
  if (std::isnan(a)) a = 14.0 / 9.0;
  if (std::isnan(bc)) bc = 1.0 / 9.0;
  if (std::isnan(h) || h <= 0.0) h = 2.0 * M_PI / (double)P.gdims[P.sd];
  if (!std::isfinite(h) || !std::isfinite(a) || !std::isfinite(bc)) return false;
  c[0] = -bc / (4.0 * h);
  c[1] = -a / (2.0 * h);
  c[2] = 0.0;
  c[3] = a / (2.0 * h);
  c[4] = bc / (4.0 * h);
  return true;
}

static ctri_status compact_loopback_group(const ctri_plan* plans, int nparts, std::vector<Plan*>* G) {
  if (!plans || nparts < 1) return fail(CTRI_ERR_INVALID_ARG, "NULL arguments");
  G->resize(nparts);
  for (int r = 0; r < nparts; ++r) {
    (*G)[r] = reinterpret_cast<Plan*>(plans[r]);
    if (!(*G)[r] || (*G)[r]->rank != r || (*G)[r]->p != nparts || !(*G)[r]->loopback)
      return fail(CTRI_ERR_INVALID_ARG, "plans must be one loopback group in rank order");
  }
  return CTRI_OK;
}

ctri_status ctri_compact_apply(ctri_plan plan, const double coef[5], const double* f, double* out,
                               ctri_stream stream) {
  if (!plan) return fail(CTRI_ERR_INVALID_ARG, "NULL plan");
  Plan* P = reinterpret_cast<Plan*>(plan);
  std::vector<Plan*> G{P};
  if (P->loopback && P->p > 1) return fail(CTRI_ERR_INVALID_ARG, "loopback plan: use ctri_compact_apply_loopback");
  return deriv_group(G, &f, &out, coef, (cudaStream_t)stream);
}

ctri_status ctri_compact_apply_loopback(const ctri_plan* plans, int nparts, const double coef[5],
                                        const double* const* f, double* const* out,
                                        ctri_stream stream) {
  std::vector<Plan*> G;
  TRY(compact_loopback_group(plans, nparts, &G));
  if (!f || !out) return fail(CTRI_ERR_INVALID_ARG, "NULL arguments");
  return deriv_group(G, f, out, coef, (cudaStream_t)stream);
}

ctri_status ctri_deriv(ctri_plan plan, const double* f, double* df, double a, double bc, double h,
                       ctri_stream stream) {
  if (!plan) return fail(CTRI_ERR_INVALID_ARG, "NULL plan");
  double c[5];
  if (!deriv_coef(*reinterpret_cast<Plan*>(plan), a, bc, h, c))
    return fail(CTRI_ERR_INVALID_ARG, "non-finite a, bc or h");
  return ctri_compact_apply(plan, c, f, df, stream);
}

ctri_status ctri_deriv_loopback(const ctri_plan* plans, int nparts, const double* const* f,
                                double* const* df, double a, double bc, double h,
                                ctri_stream stream) {
  if (!plans || nparts < 1 || !plans[0]) return fail(CTRI_ERR_INVALID_ARG, "NULL arguments");
  double c[5];
  if (!deriv_coef(*reinterpret_cast<Plan*>(plans[0]), a, bc, h, c))
    return fail(CTRI_ERR_INVALID_ARG, "non-finite a, bc or h");
  return ctri_compact_apply_loopback(plans, nparts, c, f, df, stream);
}

ctri_status ctri_scheme_coef(int scheme, double delta, double coef[5], double bands[3]) {
  double c[5] = {0, 0, 0, 0, 0}, al = 0;
  switch (scheme) {
    case CTRI_SCHEME_COLLOCATED_D1: {  // alpha = 1/3, a = 14/9, b = 1/9 (R8)
      if (!(delta > 0) || !std::isfinite(delta)) return fail(CTRI_ERR_INVALID_ARG, "delta must be > 0");
      const double a = 14.0 / 9.0, b = 1.0 / 9.0;
      c[0] = -b / (4 * delta); c[1] = -a / (2 * delta); c[3] = a / (2 * delta); c[4] = b / (4 * delta);
      al = 1.0 / 3.0;
      break;
    }
    case CTRI_SCHEME_STAGGERED_D1: {  // alpha = 9/62, a = 63/62, b = 17/62 (R18)
      if (!(delta > 0) || !std::isfinite(delta)) return fail(CTRI_ERR_INVALID_ARG, "delta must be > 0");
      const double a = 63.0 / 62.0, b = 17.0 / 62.0;
      c[0] = -b / (3 * delta); c[1] = -a / delta; c[2] = a / delta; c[3] = b / (3 * delta);
      al = 9.0 / 62.0;
      break;
    }
    case CTRI_SCHEME_STAGGERED_I: {  // alpha = 3/10, a = 3/2, b = 1/10 (R18)
      const double a = 1.5, b = 0.1;
      c[0] = b / 2; c[1] = a / 2; c[2] = a / 2; c[3] = b / 2;
      al = 0.3;
      break;
    }
    default:
      return fail(CTRI_ERR_INVALID_ARG, "unknown scheme");
  }
  if (coef) for (int k = 0; k < 5; ++k) coef[k] = c[k];
  if (bands) { bands[0] = al; bands[1] = 1.0; bands[2] = al; }
  return CTRI_OK;
}

ctri_status ctri_get_stats(ctri_plan plan, ctri_stats* out) {
  if (!plan || !out) return fail(CTRI_ERR_INVALID_ARG, "NULL argument");
  Plan* P = reinterpret_cast<Plan*>(plan);
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out->global_dims, P->gdims, sizeof(P->gdims));
  out->solve_dim = P->sd;
  out->nparts = P->p;
  out->rank = P->rank;
  out->cyclic = P->cyclic;
  out->n_local = P->lay.n;
  out->m_batch = P->lay.m();
  out->local_kernel = P->local_kernel;
  out->rows_per_thread = P->local_kernel ? P->tile.K : 0;
  out->cluster_size = P->local_kernel ? P->tile.G : 1;
  out->tile_columns = P->local_kernel ? P->tile.C : 1;
  out->tile_variant = P->local_kernel ? P->tile.variant : -1;
  out->tile_stages = P->local_kernel ? P->tile.STAGES : 0;
  out->reduced_rows = P->p * P->rvp;
  out->vchain = P->vchain ? 1 : 0;
  out->reduced_path = (P->fused || (P->p == 1 && P->vchain)) ? 3 : (P->p > 1 && P->p2p) ? ((P->allgather || (P->r == 2 && !P->ppcr)) ? 2 : 1) : 0;
  out->band_halfwidth = P->r;
  out->vparts = P->vp;
  out->grid_ctas = P->local_kernel ? P->tile.grid : (int32_t)((P->tlay.m() + 127) / 128);
  out->device_error = 0;
  if (P->h_err) {
    CUDA_TRY(cudaDeviceSynchronize());  // kernels of the last solve have stored their error words
    out->device_error = *reinterpret_cast<volatile int*>(P->h_err);
  }
  if (P->d_epoch) CUDA_TRY(cudaMemcpy(&out->p2p_epoch, P->d_epoch, sizeof(unsigned int), cudaMemcpyDeviceToHost));
  if (P->d_hepoch) CUDA_TRY(cudaMemcpy(&out->halo_epoch, P->d_hepoch, sizeof(unsigned int), cudaMemcpyDeviceToHost));
  out->chunk_heads = P->local_kernel ? P->tile.Q : 1;
  const int64_t interior = P->tlay.n - P->r;
  const bool full = (P->flags & CTRI_FLAG_FULL_BACKSUB) || (2 * P->window >= interior);
  out->window_rows = (int32_t)(full ? interior : P->window);
  out->pcr_stages = P->sched.pcr_stages;
  out->detach_stages = P->sched.detach_stages;
  out->detached_rows = P->sched.detached_rows;
  if (P->p > 1) {
    int sends = 0, rounds = 0;
    schedule_counts(*P, &sends, &rounds);
    out->comm_rounds = rounds;
    out->sends_per_solve = sends;
    out->bytes_sent_per_solve = (int64_t)sends * 8 * P->lay.m();
  }
  out->launches_per_solve = P->launches_per_solve;
  out->solves = P->solves;
  float* ts[] = {&out->t_total_us, &out->t_local_us, &out->t_yexchange_us, &out->t_bhat_us,
                 &out->t_xexchange_us, &out->t_backsub_us};
  for (float* t : ts) *t = -1.f;
  for (int k = 0; k < CTRI_MAX_STAGES; ++k) out->t_stage_us[k] = out->t_p2p_step_us[k] = -1.f;
  out->t_reduced_kernel_us = out->t_window_us = out->t_p2p_y_us = out->t_p2p_x_us = -1.f;
  if (P->timed_valid || (!P->ev.empty() && P->solves > 0)) {
    const bool two = P->p > 1 || (P->vp > 1 && !P->vchain) || P->r == 2;
    CUDA_TRY(cudaEventSynchronize(P->ev[two ? EV_BACK : EV_LOCAL]));
    out->t_local_us = elapsed(*P, EV_START, EV_LOCAL);
    if (P->p > 1 && P->p2p && !P->fused) {
      out->t_backsub_us = elapsed(*P, EV_LOCAL, EV_BACK);  // (a2)-(a4): P2P kernel + window pass
      out->t_total_us = elapsed(*P, EV_START, EV_BACK);
      out->t_reduced_kernel_us = elapsed(*P, EV_LOCAL, EV_XX);
      out->t_window_us = elapsed(*P, EV_XX, EV_BACK);
      if (P->d_trace && P->trace_ctas > 0) {  // per-round medians over the CTAs of this rank
        const int grid = P->trace_ctas;
        std::vector<unsigned long long> t((size_t)kP2PTrace * grid);
        CUDA_TRY(cudaMemcpy(t.data(), P->d_trace, t.size() * 8, cudaMemcpyDeviceToHost));
        auto med = [&](int a, int b) -> float {
          std::vector<double> v;
          for (int k = 0; k < grid; ++k) {
            const unsigned long long* tk = t.data() + (size_t)kP2PTrace * k;
            if (tk[a] && tk[b] >= tk[a]) v.push_back((double)(tk[b] - tk[a]) * 1e-3);
          }
          if (v.empty()) return -1.f;
          std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
          return (float)v[v.size() / 2];
        };
        const int q = P->r == 2 ? (P->ppcr ? P->ppcr_steps : 0)
                                : (P->allgather ? 0 : (int)P->sched.steps.size());
        out->p2p_steps = q;
        out->t_p2p_y_us = med(kTrStart, kTrYRecv);
        int prev = kTrYRecv;
        for (int k = 0; k < q && k < CTRI_MAX_STAGES; ++k) {
          out->t_p2p_step_us[k] = med(prev, kTrStep0 + k);
          prev = kTrStep0 + k;
        }
        out->t_p2p_x_us = med(prev, kTrXRecv);
      }
    } else if (P->p > 1) {
      out->t_yexchange_us = elapsed(*P, EV_LOCAL, EV_YX);
      out->t_bhat_us = elapsed(*P, EV_YX, EV_BHAT);
      int prev = EV_BHAT;
      for (int k = 0; k < P->gpcr.stages; ++k) {
        out->t_stage_us[k] = elapsed(*P, prev, EV_STAGE0 + k);
        prev = EV_STAGE0 + k;
      }
      out->t_xexchange_us = elapsed(*P, prev, EV_XX);
      out->t_backsub_us = elapsed(*P, EV_XX, EV_BACK);
      out->t_total_us = elapsed(*P, EV_START, EV_BACK);
    } else if ((P->vp > 1 && !P->vchain) || P->r == 2) {
      out->t_backsub_us = elapsed(*P, EV_LOCAL, EV_BACK);  // local reduced + window back-sub
      out->t_total_us = elapsed(*P, EV_START, EV_BACK);
    } else {
      out->t_total_us = out->t_local_us;
    }
  }
  return CTRI_OK;
}

ctri_status ctri_plan_destroy(ctri_plan plan) {
  if (!plan) return CTRI_OK;
  Plan* P = reinterpret_cast<Plan*>(plan);
  // detach from a loopback group
  for (Plan* q : P->group)
    if (q && q != P)
      for (auto& g : q->group)
        if (g == P) g = nullptr;
  free_plan(P);
  return CTRI_OK;
}

ctri_status ctri_factor_query(int64_t n, const double bands[3], double* S, double* R, double* hat,
                              int* window) {
  if (!bands) return fail(CTRI_ERR_INVALID_ARG, "NULL bands");
  if (n < 3) return fail(CTRI_ERR_PARTITION_TOO_SMALL, "n < 3");
  Partition pt;
  FactorError fe;
  if (!partition_factor(n - 1, Bands{bands[0], bands[1], bands[2]}, &pt, &fe))
    return fail((ctri_status)fe.code, fe.detail);
  if (S) std::memcpy(S, pt.S.data(), sizeof(double) * (n - 1));
  if (R) std::memcpy(R, pt.R.data(), sizeof(double) * (n - 1));
  if (hat) {
    hat[0] = pt.Lh;
    hat[1] = pt.Dh;
    hat[2] = pt.Uh;
  }
  if (window) *window = (int)backsub_window(pt);
  return CTRI_OK;
}

ctri_status ctri_pcr_coefficients(int P, int cyclic, const double* L, const double* D,
                                  const double* U, double* alpha, double* gamma, double* inv,
                                  int* stages) {
  if (P < 1 || !L || !D || !U || !inv || !stages) return fail(CTRI_ERR_INVALID_ARG, "bad arguments");
  PcrTables t;
  FactorError fe;
  double mx = 0;
  for (int c = 0; c < P; ++c) mx = std::max(mx, std::max(std::fabs(D[c]), std::max(std::fabs(L[c]), std::fabs(U[c]))));
  if (!pcr_factor(P, cyclic != 0, std::vector<double>(L, L + P), std::vector<double>(D, D + P),
                  std::vector<double>(U, U + P), 1e-13 * mx, &t, &fe))
    return fail((ctri_status)fe.code, fe.detail);
  *stages = t.stages;
  if (alpha) std::memcpy(alpha, t.alpha.data(), sizeof(double) * t.alpha.size());
  if (gamma) std::memcpy(gamma, t.gamma.data(), sizeof(double) * t.gamma.size());
  std::memcpy(inv, t.inv.data(), sizeof(double) * P);
  return CTRI_OK;
}

ctri_status ctri_reduced_schedule(int P, int cyclic, const double* L, const double* D,
                                  const double* U, int max_steps, int* nsteps, int* kinds,
                                  double* w, int* src, double* c, int* counts) {
  if (P < 1 || !L || !D || !U || !nsteps || !kinds || !w || !src || !c || !counts)
    return fail(CTRI_ERR_INVALID_ARG, "bad arguments");
  double mx = 0;
  for (int i = 0; i < P; ++i)
    mx = std::max(mx, std::max(std::fabs(D[i]), std::max(std::fabs(L[i]), std::fabs(U[i]))));
  Schedule sc;
  FactorError fe;
  if (!reduced_schedule(P, cyclic != 0, std::vector<double>(L, L + P), std::vector<double>(D, D + P),
                        std::vector<double>(U, U + P), 1e-13 * mx, &sc, &fe))
    return fail((ctri_status)fe.code, fe.detail);
  const int ns = (int)sc.steps.size();
  if (ns > max_steps) return fail(CTRI_ERR_INVALID_ARG, "max_steps too small");
  *nsteps = ns;
  for (int s = 0; s < ns; ++s) {
    kinds[s] = sc.kind[s];
    for (int i = 0; i < P; ++i) {
      const SchedEntry& e = sc.steps[s][i];
      w[(size_t)s * P + i] = e.w;
      for (int k = 0; k < 2; ++k) {
        src[2 * ((size_t)s * P + i) + k] = e.src[k];
        c[2 * ((size_t)s * P + i) + k] = e.c[k];
      }
    }
  }
  counts[0] = sc.pcr_stages;
  counts[1] = sc.detach_stages;
  counts[2] = sc.detached_rows;
  return CTRI_OK;
}

ctri_status ctri_penta_factor_query(int64_t n, const double bands[5], double* SR, double* hat,
                                   int* window) {
  if (!bands || !SR || !hat || !window) return fail(CTRI_ERR_INVALID_ARG, "NULL argument");
  Penta pt;
  FactorError fe;
  if (!penta_factor(n - 2, bands, &pt, &fe)) return fail((ctri_status)fe.code, fe.detail);
  const int64_t N = n - 2;
  const std::vector<double>* v[4] = {&pt.S0, &pt.S1, &pt.R0, &pt.R1};
  for (int k = 0; k < 4; ++k) std::memcpy(SR + k * N, v[k]->data(), sizeof(double) * N);
  std::memcpy(hat, pt.Lh, sizeof(pt.Lh));
  std::memcpy(hat + 4, pt.Dh, sizeof(pt.Dh));
  std::memcpy(hat + 8, pt.Uh, sizeof(pt.Uh));
  std::memcpy(hat + 12, pt.DhFirst, sizeof(pt.DhFirst));
  *window = (int)penta_window(pt);
  return CTRI_OK;
}

ctri_status ctri_penta_block_pcr(int P, int cyclic, int64_t n, const double bands[5], int max_stages,
                                 double* alpha, double* gamma, double* fold, int* stages) {
  if (!bands || !alpha || !gamma || !fold || !stages) return fail(CTRI_ERR_INVALID_ARG, "NULL argument");
  Penta pt;
  FactorError fe;
  if (!penta_factor(n - 2, bands, &pt, &fe)) return fail((ctri_status)fe.code, fe.detail);
  double mx = 0;
  for (int k = 0; k < 5; ++k) mx = std::max(mx, std::fabs(bands[k]));
  PentaPcr t;
  if (!penta_block_pcr(P, cyclic != 0, pt, 1e-13 * mx, &t, &fe)) return fail((ctri_status)fe.code, fe.detail);
  if (t.stages > max_stages) return fail(CTRI_ERR_INVALID_ARG, "max_stages too small");
  std::memcpy(alpha, t.alpha.data(), sizeof(double) * t.alpha.size());
  std::memcpy(gamma, t.gamma.data(), sizeof(double) * t.gamma.size());
  std::memcpy(fold, t.fold.data(), sizeof(double) * t.fold.size());
  *stages = t.stages;
  return CTRI_OK;
}

ctri_status ctri_penta_reduced_schedule_apply(int P, int cyclic, int64_t n, const double bands[5],
                                              const double* bhat, double* xt, int* steps,
                                              int* detach_stages, int* detached_rows) {
  if (P < 1 || !bands || !bhat || !xt) return fail(CTRI_ERR_INVALID_ARG, "bad arguments");
  Penta pt;
  FactorError fe;
  if (!penta_factor(n - 2, bands, &pt, &fe)) return fail((ctri_status)fe.code, fe.detail);
  double mx = 0;
  for (int k = 0; k < 5; ++k) mx = std::max(mx, std::fabs(bands[k]));
  BlockSchedule sc;
  if (!penta_reduced_schedule(P, cyclic != 0, pt, 1e-13 * mx, &sc, &fe)) return fail((ctri_status)fe.code, fe.detail);
  std::vector<double> v(bhat, bhat + 2 * P);
  for (const auto& st : sc.steps) {  // every row reads its sources' pre-step values
    std::vector<double> nv = v;
    for (int i = 0; i < P; ++i) {
      const BlockSchedEntry& e = st[i];
      double r0 = e.W[0] * v[2 * i] + e.W[1] * v[2 * i + 1];
      double r1 = e.W[2] * v[2 * i] + e.W[3] * v[2 * i + 1];
      for (int k = 0; k < 2; ++k) {
        if (e.src[k] < 0) continue;
        const double u0 = v[2 * e.src[k]], u1 = v[2 * e.src[k] + 1];
        r0 -= e.C[k][0] * u0 + e.C[k][1] * u1;
        r1 -= e.C[k][2] * u0 + e.C[k][3] * u1;
      }
      nv[2 * i] = r0;
      nv[2 * i + 1] = r1;
    }
    v.swap(nv);
  }
  std::memcpy(xt, v.data(), sizeof(double) * 2 * P);
  if (steps) *steps = (int)sc.steps.size();
  if (detach_stages) *detach_stages = sc.detach_stages;
  if (detached_rows) *detached_rows = sc.detached_rows;
  return CTRI_OK;
}

ctri_status ctri_reduced_inverse(int P, int cyclic, const double* L, const double* D,
                                 const double* U, double* inv) {
  if (P < 1 || !L || !D || !U || !inv) return fail(CTRI_ERR_INVALID_ARG, "bad arguments");
  double mx = 0;
  for (int i = 0; i < P; ++i)
    mx = std::max(mx, std::max(std::fabs(D[i]), std::max(std::fabs(L[i]), std::fabs(U[i]))));
  std::vector<double> out;
  FactorError fe;
  if (!reduced_inverse(P, cyclic != 0, std::vector<double>(L, L + P), std::vector<double>(D, D + P),
                       std::vector<double>(U, U + P), 1e-13 * mx, &out, &fe))
    return fail((ctri_status)fe.code, fe.detail);
  std::memcpy(inv, out.data(), sizeof(double) * out.size());
  return CTRI_OK;
}

}  // extern "C"
