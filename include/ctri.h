/*
 * ctri.h -- C ABI of the B200-native batched cyclic tridiagonal solver.
 *
 * The library solves A x = b for every batch column of a 3D right-layout
 * grid (third index contiguous, "right memory layout is used,
 * where the third index maps to contiguous memory"), A the cyclic (or
 * acyclic) tridiagonal matrix with constant bands (l, d, u) =
 * (A[i,i-1], A[i,i], A[i,i+1]); cyclic corners A[0,N-1] = l, A[N-1,0] = u.
 * The benchmark matrix is B[1/3, 1, 1/3] (P:5).
 *
 * The solve direction is sharded over `nparts` ranks (one GPU each), rank i
 * owning global rows [i*n, (i+1)*n), n = N/nparts (P:5 "the domain is
 * decomposed equally along the solving direction").  Local row 0 of every
 * slab is the interface unknown x~_i, rows 1..n-1 the interior x_i
 * (Eqs. system1/system2; reading R1).  Per solve the
 * library runs the paper's method (Sec. "Parallel linear solver"):
 *   (a1) y_i = D_i^{-1} b_i on every column (Eq. yi; per-partition PCR),
 *   (a2) b^_i = b~_i - L~_i y_{i-1} - U~_i y_i (Eq. bi_hat), one exchange i -> i+1,
 *   (a3) cyclic PCR on the reduced system A^ x~ = b^ in log2(nparts) pairwise
 *        stages with partners i +- 2^k,
 *   (a4) x_i = y_i - S_i x~_i - R_i x~_{i+1} (Eq. xi_app), one exchange i+1 -> i.
 * Everything that does not depend on b (S_i, R_i, L^, D^, U^, the per-stage
 * reduction coefficients) is pre-factorised at plan creation.
 *
 * Conventions for every entry point:
 *  - Return a ctri_status; no exception crosses the ABI.  On failure a
 *    thread-local detail string is available from ctri_last_error().
 *  - Device pointers are CUDA device addresses on the current device, fp64,
 *    16-byte aligned, holding the LOCAL slab in right layout with local dims
 *    = global dims except dims[solve_dim] = N/nparts.  The caller owns them.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Solves are
 *    asynchronous and stream ordered; with nparts > 1 they are collective:
 *    every rank calls with the same plan parameters in the same order.
 */
#ifndef CTRI_H
#define CTRI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTRI_ABI_VERSION 6

typedef struct ctri_plan_s* ctri_plan;
typedef struct CUstream_st* ctri_stream; /* == cudaStream_t */

typedef enum ctri_status {
  CTRI_OK = 0,
  CTRI_ERR_INVALID_ARG = 1,     /* bad pointer, dims, solve_dim, rank, alignment */
  CTRI_ERR_UNSUPPORTED = 2,     /* e.g. cyclic non-power-of-two nparts with CTRI_FLAG_NCCL_ROUNDS */
  CTRI_ERR_SINGULAR = 3,        /* plan-time pivot guard: |pivot| < 1e-13 * max|band| */
  CTRI_ERR_PARTITION_TOO_SMALL = 4, /* n = N/nparts < 3 or N not divisible by nparts */
  CTRI_ERR_CUDA = 5,            /* a CUDA runtime call or kernel launch failed */
  CTRI_ERR_NCCL = 6,            /* an NCCL call failed */
  CTRI_ERR_OOM = 7              /* device or pinned-host allocation failed */
} ctri_status;

/* Plan flags (bitwise OR). */
#define CTRI_FLAG_FULL_BACKSUB   (1u << 0) /* (a4) on every interior row instead of the window W (R15) */
#define CTRI_FLAG_GENERIC_LOCAL  (1u << 1) /* force the column-serial local-solve kernel (testing) */
#define CTRI_FLAG_TIMING         (1u << 2) /* record per-phase CUDA events; read with ctri_get_stats */
#define CTRI_FLAG_DERIV          (1u << 3) /* allocate halo planes so ctri_deriv may be called */
#define CTRI_FLAG_NCCL_ROUNDS    (1u << 4) /* nparts > 1: host-issued NCCL rounds instead of the fused
                                              device-initiated P2P reduced phase */
#define CTRI_FLAG_FUSED_REDUCED  (1u << 6) /* 2 <= nparts <= 8, real GPUs (not loopback), strided
                                              tile path: run (a2)-(a4) INSIDE the local-solve tile
                                              kernel (window rows kept on chip, planes all-gathered
                                              as LL words, finalised one tile later).  Opt-in: on
                                              B200 it measures slower than the separate P2P kernel
                                              + window pass.  Ignored where
                                              it does not apply. */
#define CTRI_FLAG_ALLGATHER      (1u << 5) /* 2 <= nparts <= 8, P2P path: solve the reduced system with
                                              ONE all-gather round of 2 planes per rank and plan-time
                                              rows of A^{-1} (latency comparison for
                                              the log2 p pairwise stages).  UNSUPPORTED otherwise. */

#define CTRI_MAX_STAGES 16

typedef struct ctri_stats {
  int64_t global_dims[3];
  int32_t solve_dim, nparts, rank, cyclic;
  int64_t n_local;              /* rows of the local slab along solve_dim */
  int64_t m_batch;              /* batch columns = product of the two other dims */
  int32_t local_kernel;         /* 0 = column-serial, 1 = cluster-tile (strided axis), 2 = cluster-tile (contiguous axis) */
  int32_t rows_per_thread;      /* K of the tile kernel (0 for column-serial) */
  int32_t cluster_size;         /* CTAs cooperating on one column tile */
  int32_t tile_columns;         /* batch columns per tile */
  int32_t chunk_heads;          /* Q: on-chip reduced-system rows per column */
  int32_t window_rows;          /* W: rows per slab end touched by (a4); n-1 means all rows */
  int32_t pcr_stages;           /* q = log2(nparts) distributed PCR stages */
  int32_t comm_rounds;          /* dependent exchange rounds per solve: 2 + q (nparts > 1) */
  int32_t sends_per_solve;      /* messages sent by this rank per solve: 2q + 1 */
  int64_t bytes_sent_per_solve; /* 8 m * sends */
  int32_t launches_per_solve;   /* kernels this library launches per ctri_solve */
  uint64_t solves;              /* ctri_solve calls on this plan */
  /* Per-phase device times of the LAST solve in microseconds (CTRI_FLAG_TIMING; else -1).
     ctri_get_stats synchronises the plan's events. */
  float t_total_us, t_local_us, t_yexchange_us, t_bhat_us;
  float t_stage_us[CTRI_MAX_STAGES]; /* exchange + update of PCR stage k */
  float t_xexchange_us, t_backsub_us;
  int32_t tile_variant;         /* cluster-tile variant index (columns/threads/ring depth), -1 if none */
  int32_t tile_stages;          /* TMA shared-memory ring depth of the tile kernel */
  int32_t reduced_path;         /* nparts > 1: 0 = NCCL rounds, 1 = fused P2P kernel (t_backsub_us
                                   then times the whole fused (a2)-(a4) kernel), 2 = P2P all-gather,
                                   3 = fused into the local-solve tile kernel (t_local_us = all);
                                   nparts == 1 with vparts > 1: 3 when the virtual partitions'
                                   reduced system and window rows are finished inside the
                                   tile kernel (default), else 0 (k_reduced_local + k_window) */
  int32_t device_error;         /* nonzero: a P2P wait hit its deadline (peer missing) */
  int32_t vparts;               /* nparts == 1: partitions of the slab solved on this GPU (the
                                   paper's partition method; (a2)-(a4) then run on-device) */
  int32_t grid_ctas;            /* CTAs of the local-solve launch */
  int32_t detach_stages;        /* nparts > 1 cyclic, not a power of two: detach stages */
  int32_t detached_rows;        /* rows detached and reattached: nparts - 2^floor(log2 nparts) */
  int32_t band_halfwidth;       /* r: 1 tridiagonal plan, 2 pentadiagonal plan */
  /* device-initiated reduced phase (reduced_path 1 / 2, CTRI_FLAG_TIMING): CUDA-event times of
     the P2P kernel and of the window kernel, and per-round medians over the kernel's CTAs of
     %globaltimer stamps (y round incl. waiting for the left neighbour, each schedule step, x~
     round); -1 where not applicable */
  float t_reduced_kernel_us, t_window_us;
  float t_p2p_y_us, t_p2p_step_us[CTRI_MAX_STAGES], t_p2p_x_us;
  int32_t p2p_steps;            /* schedule steps timed in t_p2p_step_us */
  uint32_t p2p_epoch;           /* device epoch of the reduced-phase mailboxes (slice 0): one per
                                   solve, so its parity alternates the double-buffered copies */
  int32_t reduced_rows;         /* rows of the reduced system this solve exchanges across ranks:
                                   nparts (one per rank; with vparts > 1 the virtual partitions
                                   are chained inside the tile kernel) or nparts * vparts ("virtual
                                   rows", each its own row of the distributed PCR) */
  int32_t vchain;               /* 1: the virtual partitions' reduced system and window rows are
                                   finished inside the tile kernel (the virtual-partition chain) */
  uint32_t halo_epoch;          /* device epoch of the derivative halo exchange (slice 0): one per
                                   ctri_deriv / ctri_compact_apply, independent of p2p_epoch */
} ctri_stats;

/* Human-readable status name; never NULL. */
const char* ctri_status_string(ctri_status s);

/* Detail of the last failure on the calling thread ("" if none). */
const char* ctri_last_error(void);

/* ABI version (CTRI_ABI_VERSION) -- lets the binding check it loaded the right library. */
int ctri_abi_version(void);

/* Fill `out` (128 bytes) with a fresh NCCL unique id.  Rank 0 calls this and
 * broadcasts the bytes (the Python binding uses torch.distributed) before
 * every rank calls ctri_plan_create. */
ctri_status ctri_get_unique_id(void* out128);

/* Create a plan (pre-factorisation) for this rank.
 *   global_dims  [3] global grid dims, right layout.
 *   solve_dim    0, 1 or 2: index along which every column is solved.
 *   nparts       partitions of the solve direction == ranks; rank in [0, nparts).
 *   bands        {l, d, u}; constant along the solve direction.
 *   cyclic       1 periodic (the paper's benchmark), 0 acyclic.
 *   nccl_unique_id  128-byte ncclUniqueId shared by all ranks; NULL iff nparts == 1.
 *   flags        CTRI_FLAG_*.
 *   stream       stream used for the table uploads during create.
 * Errors: INVALID_ARG, PARTITION_TOO_SMALL, UNSUPPORTED (cyclic non-power-of-two nparts on the
 * NCCL-rounds path, or cyclic non-power-of-two nparts > 16 = kMaxP2PRanks on the P2P path),
 * SINGULAR (pivot guard), CUDA, NCCL, OOM.  On error *out is NULL.
 * The plan owns its device tables, plane buffers, events and NCCL communicator. */
ctri_status ctri_plan_create(ctri_plan* out, const int64_t global_dims[3], int solve_dim,
                             int nparts, int rank, const double bands[3], int cyclic,
                             const void* nccl_unique_id, uint32_t flags, ctri_stream stream);

/* TEST-ONLY in-process "loopback" group: create `nparts` plans on the current
 * device (ranks 0..nparts-1) whose exchanges are device-to-device copies
 * instead of NCCL messages.  Solve them together with ctri_solve_loopback.
 * `plans` receives nparts handles; destroy each with ctri_plan_destroy. */
ctri_status ctri_plan_create_loopback(ctri_plan* plans, int nparts, const int64_t global_dims[3],
                                      int solve_dim, const double bands[3], int cyclic,
                                      uint32_t flags, ctri_stream stream);

/* PENTADIAGONAL plan (r = 2; "for a penta-diagonal system (w = 5), D~_i is
 * 2x2").  bands = {e, l, d, u, f} = A[i,i-2], A[i,i-1], A[i,i], A[i,i+1],
 * A[i,i+2] (host array, copied); cyclic wraps the four corner couplings.  Each of the nparts
 * slabs keeps two interface rows (local rows 0, 1) and n - 2 >= 4 interior rows; the 2x2-block
 * reduced system is solved over the P2P mailboxes by its 2x2-block step schedule (P:346 with
 * 2x2 blocks, R20: a y round, the block PCR steps -- with block detach / reattach
 * for cyclic non-power-of-two nparts, P:271 / P:294 -- the fold, an x~ round) or, with
 * CTRI_FLAG_ALLGATHER, by ONE all-gather round and plan-time rows of its inverse (nparts <= 8).
 * The local solve runs on chip (2x2-block PCR of 32-row chunk heads in thread-block clusters)
 * for strided slabs of 256..2048 rows, and for longer strided slabs (n a power-of-two multiple
 * of 1024, at most 8 of them) as n/1024 partitions of one GPU: with nparts == 1 their reduced
 * system is solved on the GPU, with nparts > 1 (solve index 0, nparts * n/1024 <= 16, not
 * CTRI_FLAG_ALLGATHER) they become virtual block rows of the distributed reduced system
 * (rows of one GPU exchange through its own mailbox; ctri_get_stats reports vparts and
 * reduced_rows); column-serial otherwise (contiguous axis, other sizes).  b and x must be
 * 16-byte aligned (INVALID_ARG otherwise).
 * The plan is used with ctri_solve / ctri_solve_loopback / ctri_solve_host /
 * ctri_get_stats / ctri_plan_destroy like a tridiagonal one.  Errors: INVALID_ARG (as
 * ctri_plan_create), PARTITION_TOO_SMALL (n < 6 or N % nparts), UNSUPPORTED (nparts > 8,
 * CTRI_FLAG_NCCL_ROUNDS, CTRI_FLAG_DERIV or CTRI_FLAG_GENERIC_LOCAL), SINGULAR (pivot guard
 * 1e-13 * max|band| in the interior LU or the reduced inverse). */
ctri_status ctri_plan_create_penta(ctri_plan* out, const int64_t global_dims[3], int solve_dim,
                                   int nparts, int rank, const double bands[5], int cyclic,
                                   const void* nccl_unique_id, uint32_t flags, ctri_stream stream);

/* TEST-ONLY: a pentadiagonal loopback group on the current device (see
 * ctri_plan_create_loopback). */
ctri_status ctri_plan_create_penta_loopback(ctri_plan* plans, int nparts,
                                            const int64_t global_dims[3], int solve_dim,
                                            const double bands[5], int cyclic, uint32_t flags,
                                            ctri_stream stream);

/* Solve on device buffers: x = A^{-1} b for the local slab.  x == b (in place) is
 * allowed; partial overlap is not.  Asynchronous, stream ordered, collective.
 * Errors: INVALID_ARG (NULL/misaligned), CUDA, NCCL. */
ctri_status ctri_solve(ctri_plan plan, const double* b, double* x, ctri_stream stream);

/* Solve a loopback group: b[r], x[r] are rank r's slabs (device pointers). */
ctri_status ctri_solve_loopback(const ctri_plan* plans, int nparts, const double* const* b,
                                double* const* x, ctri_stream stream);

/* End-to-end solve from HOST memory: copies b_host to the device, solves and copies
 * the result back into x_host, all on `stream` (pinned host memory gives
 * asynchronous DMA; pageable memory works but blocks).  The plan allocates its
 * device staging slab on first use.  Returns after enqueuing; synchronise the
 * stream before reading x_host. */
ctri_status ctri_solve_host(ctri_plan plan, const double* b_host, double* x_host,
                            ctri_stream stream);

/* Compact first derivative along solve_dim:
 *   rhs_j = a (f_{j+1}-f_{j-1})/(2h) + bc (f_{j+2}-f_{j-2})/(4h)  (periodic, halo from
 *   ranks i-1 / i+1), then df = A^{-1} rhs with this plan's bands.
 * Defaults (the library fills them in, so callers carry no scheme arithmetic):
 *   a or bc NaN  -> Lele's sixth-order pair a = 14/9, bc = 1/9 (the paper prints only the
 *                   symbols; reading R8);
 *   h <= 0 or NaN -> h = 2 pi / N_global[solve_dim] (periodic domain [0, 2 pi)).
 * Requires a cyclic plan created with CTRI_FLAG_DERIV and n >= 2.  f and df must not
 * overlap.  Asynchronous, stream ordered, collective. */
ctri_status ctri_deriv(ctri_plan plan, const double* f, double* df, double a, double bc,
                       double h, ctri_stream stream);

/* TEST-ONLY: ctri_deriv for a loopback group (f[r], df[r] are rank r's slabs). */
ctri_status ctri_deriv_loopback(const ctri_plan* plans, int nparts, const double* const* f,
                                double* const* df, double a, double bc, double h,
                                ctri_stream stream);

/* A compact scheme with a five-point periodic right-hand side:
 *   rhs_j = sum_{k=-2..2} coef[k+2] f_{j+k}   (indices along solve_dim; periodic, halo
 *   planes from ranks i-1 / i+1),   out = A^{-1} rhs with this plan's bands.
 * Covers the collocated derivative above (coef = {-bc/4h, -a/2h, 0, a/2h, bc/4h}) and the
 * staggered sixth-order derivative and interpolation of PAPER.md P:202-206, whose half-node
 * inputs f_{i+1/2} are stored at index i:
 *   derivative    bands (9/62, 1, 9/62), coef = {-17/(186D), -63/(62D), 63/(62D), 17/(186D), 0}
 *   interpolation bands (3/10, 1, 3/10), coef = {1/20, 3/4, 3/4, 1/20, 0}.
 * coef is a host array of 5 finite doubles (copied; the caller keeps ownership).  Same
 * plan requirements, aliasing rules and ordering as ctri_deriv; CTRI_ERR_INVALID_ARG for a
 * NULL or non-finite coef. */
ctri_status ctri_compact_apply(ctri_plan plan, const double coef[5], const double* f, double* out,
                               ctri_stream stream);

/* Coefficients of the compact schemes the paper uses, computed in the library so that
 * bindings only marshal (PAPER.md P:65-67 collocated, P:202-206 staggered):
 *   scheme CTRI_SCHEME_COLLOCATED_D1  bands (1/3, 1, 1/3),  coef {-1/(36D), -7/(9D), 0, 7/(9D), 1/(36D)}
 *                                     (a = 14/9, b = 1/9 of P:66, D = grid spacing)
 *   scheme CTRI_SCHEME_STAGGERED_D1   bands (9/62, 1, 9/62), coef {-17/(186D), -63/(62D), 63/(62D), 17/(186D), 0}
 *   scheme CTRI_SCHEME_STAGGERED_I    bands (3/10, 1, 3/10), coef {1/20, 3/4, 3/4, 1/20, 0}
 * (staggered inputs f_{i+1/2} stored at index i, R18).  delta is the grid spacing
 * (ignored by the interpolation scheme; must be finite and > 0 otherwise).  coef[5] and
 * bands[3] are caller-owned host arrays; either may be NULL.  Errors: INVALID_ARG for an
 * unknown scheme or a bad delta.  Host only. */
#define CTRI_SCHEME_COLLOCATED_D1 0
#define CTRI_SCHEME_STAGGERED_D1  1
#define CTRI_SCHEME_STAGGERED_I   2
ctri_status ctri_scheme_coef(int scheme, double delta, double coef[5], double bands[3]);

/* TEST-ONLY: ctri_compact_apply for a loopback group. */
ctri_status ctri_compact_apply_loopback(const ctri_plan* plans, int nparts, const double coef[5],
                                        const double* const* f, double* const* out,
                                        ctri_stream stream);

/* Copy the plan's configuration, counters and (with CTRI_FLAG_TIMING) last-solve
 * phase times into *out.  Synchronises the plan's timing events. */
ctri_status ctri_get_stats(ctri_plan plan, ctri_stats* out);

/* Release everything the plan owns (including its NCCL communicator).  NULL is a no-op. */
ctri_status ctri_plan_destroy(ctri_plan plan);

/* ---- Host-only pre-factorisation queries (no device needed; used by the CPU tests) ---- */

/* Partition tables of one slab of n rows:
 *   S, R       [n-1] each: D S = l e_0, D R = u e_{n-2} (Eqs. Si, Ri), D the acyclic
 *              (n-1)x(n-1) interior block; NULL to skip.
 *   hat        [3]: {L^, D^, U^} of Eqs. Li_hat, Di_hat, Ui_hat; NULL to skip.
 *   window     rows per slab end that (a4) touches (R15); NULL to skip.
 * Errors: INVALID_ARG, PARTITION_TOO_SMALL, SINGULAR. */
ctri_status ctri_factor_query(int64_t n, const double bands[3], double* S, double* R,
                              double* hat, int* window);

/* Reduction coefficients of PCR on a P-row (block size 1) tridiagonal system with
 * row coefficients L[c] (on row c-1), D[c], U[c] (on row c+1); cyclic wraps indices,
 * acyclic ignores L[0] and U[P-1].  Stage k (stride s = 2^k), row c:
 *     b[c] <- b[c] - alpha[k*P+c] * b[c-s] - gamma[k*P+c] * b[c+s]
 * and after the last stage x[c] = inv[c] * b[c] (the cyclic wrap folded into the
 * diagonal, R3).  *stages = log2 P (cyclic; P must be a power of two) or
 * ceil(log2 P) (acyclic).  alpha/gamma hold stages*P entries (CTRI_MAX_STAGES*P suffices).
 * Errors: INVALID_ARG, UNSUPPORTED (cyclic non-power-of-two), SINGULAR. */
ctri_status ctri_pcr_coefficients(int P, int cyclic, const double* L, const double* D,
                                  const double* U, double* alpha, double* gamma, double* inv,
                                  int* stages);

/* Reduced-system schedule of nparts = P rows (one per rank): power-of-two cyclic and all acyclic
 * systems use PCR; cyclic systems of any other dimension use the paper's
 * detach / PCR / fold / reattach procedure (worked 11x11 example P:294).  Step s, row i:
 *     v_i <- w[s*P+i] v_i - c[2(s*P+i)] v_{src[2(s*P+i)]} - c[2(s*P+i)+1] v_{src[2(s*P+i)+1]}
 * with synchronous semantics (src = -1: no term); v starts as b^ and ends as x~.
 * kinds[s]: 0 detach, 1 PCR, 2 fold, 3 reattach.  counts[3] = {PCR stages, detach stages,
 * detached rows}.  Arrays hold max_steps*P (w) and 2*max_steps*P (src, c) entries.
 * Errors: INVALID_ARG (sizes, max_steps too small), SINGULAR (pivot guard). */
ctri_status ctri_reduced_schedule(int P, int cyclic, const double* L, const double* D,
                                  const double* U, int max_steps, int* nsteps, int* kinds,
                                  double* w, int* src, double* c, int* counts);

/* Host-only pentadiagonal partition tables for a slab of n rows (n >= 6, interior N = n - 2):
 * SR[4*N] = columns S0 | S1 | R0 | R1 (S = D^{-1} L, R = D^{-1} U, Eqs. Si/Ri with r = 2),
 * hat[16] = 2x2 row-major blocks L^ | D^ | U^ | D^ of an acyclic first partition, window = rows
 * per end of the back-substitution window (2^-64 reading).  SINGULAR on the pivot guard. */
ctri_status ctri_penta_factor_query(int64_t n, const double bands[5], double* SR, double* hat,
                                   int* window);

/* Host-only: the 2x2-block PCR tables of the pentadiagonal reduced system (P partitions of n
 * rows, cyclic P a power of two, acyclic any P >= 2): alpha / gamma [stages][P][4] and the final
 * fold / diagonal inverse [P][4], row-major 2x2 (factor.h PentaPcr).  Arrays hold
 * max_stages*P*4 (alpha, gamma) and P*4 (fold) doubles.  UNSUPPORTED for cyclic
 * non-power-of-two P. */
ctri_status ctri_penta_block_pcr(int P, int cyclic, int64_t n, const double bands[5], int max_stages,
                                 double* alpha, double* gamma, double* fold, int* stages);

/* Dense inverse of the P x P reduced matrix A^ (bands L, D, U per row; cyclic corners;
 * couplings that coincide for P <= 2 add up) into inv[P*P], row-major: the plan-time table of
 * the all-gather reduced solve (CTRI_FLAG_ALLGATHER).  Gauss-Jordan with
 * partial pivoting; SINGULAR if a pivot falls below 1e-13 * max|coefficient|. */
ctri_status ctri_reduced_inverse(int P, int cyclic, const double* L, const double* D,
                                 const double* U, double* inv);

/* HOST query (no device work): the pentadiagonal reduced system of P partitions of n rows
 * (bands as ctri_plan_create_penta) solved by its step schedule -- 2x2-block PCR, or for
 * cyclic non-power-of-two P the block detach / PCR / fold / reattach of P:271 / P:294 --
 * applied serially to bhat[2P] (row-major: row i, component c at 2i + c) into xt[2P], exactly
 * as the P2P kernel executes it rank by rank.  *steps, *detach_stages and *detached_rows
 * (each may be NULL) receive the schedule's counts.  Errors: INVALID_ARG, SINGULAR. */
ctri_status ctri_penta_reduced_schedule_apply(int P, int cyclic, int64_t n, const double bands[5],
                                              const double* bhat, double* xt, int* steps,
                                              int* detach_stages, int* detached_rows);

#ifdef __cplusplus
}
#endif
#endif /* CTRI_H */
