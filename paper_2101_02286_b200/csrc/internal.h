// internal.h -- plan object and kernel launcher declarations (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/ctri.h"
#include "factor.h"

namespace ctri {

constexpr int kMaxCluster = 8;               // portable thread-block cluster size
constexpr int kMaxClusterNonPortable = 16;  // opt-in (cudaFuncAttributeNonPortableClusterSizeAllowed)

// Layout of a local slab viewed as (outer, n, inner): element (o, r, c) at (o*n + r)*inner + c.
struct Layout {
  int64_t outer = 1, n = 0, inner = 1;
  __host__ __device__ int64_t m() const { return outer * inner; }
  __host__ __device__ int64_t elems() const { return outer * n * inner; }
};

// Parameters of the cluster-tile kernel that live in the kernel's constant bank.
template <int K>
struct TileConsts {
  double l, u;
  double inv_den[K > 1 ? K - 1 : 1];  // Thomas on the (K-1)-row chunk interior
  double mlid[K > 1 ? K - 1 : 1];     // -l * inv_den
  double cp[K > 1 ? K - 1 : 1];
  double S[K > 1 ? K - 1 : 1];        // chunk-level S_K = D_K^{-1} l e_0
  double R[K > 1 ? K - 1 : 1];        // chunk-level R_K = D_K^{-1} u e_last
};

constexpr int kMaxUniformStages = 12;  // head-system PCR stages passed as kernel parameters

// Five-point periodic RHS of a compact scheme, b_j = sum_{k=-2..2} c_k f_{j+k} (P:65-67 collocated
// derivative; P:202-206 staggered derivative / interpolation).  The three schemes of the paper are
// pair forms that keep the exact differences / sums of their definitions and cost 2 FMAs:
//   kind 1  c = (-q, -p, 0, p, q):    p (f_1 - f_-1) + q (f_2 - f_-2)    collocated derivative
//   kind 2  c = (-q, -p, p, q, 0):    p (f_0 - f_-1) + q (f_1 - f_-2)    staggered derivative
//   kind 3  c = (q, p, p, q, 0):      p (f_0 + f_-1) + q (f_1 + f_-2)    staggered interpolation
//   kind 0  anything else:            sum_k c_k f_k (5 FMAs)
struct Stencil5 {
  double c[5] = {0, 0, 0, 0, 0};
  double p = 0, q = 0;
  int kind = 0;
};
inline Stencil5 make_stencil5(const double c[5]) {
  Stencil5 s;
  for (int k = 0; k < 5; ++k) s.c[k] = c[k];
  if (c[2] == 0.0 && c[1] == -c[3] && c[0] == -c[4]) {
    s.kind = 1, s.p = c[3], s.q = c[4];
  } else if (c[4] == 0.0 && c[1] == -c[2] && c[0] == -c[3]) {
    s.kind = 2, s.p = c[2], s.q = c[3];
  } else if (c[4] == 0.0 && c[1] == c[2] && c[0] == c[3]) {
    s.kind = 3, s.p = c[2], s.q = c[3];
  }
  return s;
}
// v0..v4 = f_{j-2} .. f_{j+2}
__host__ __device__ __forceinline__ double apply_stencil5(const Stencil5& s, double v0, double v1,
                                                          double v2, double v3, double v4) {
  switch (s.kind) {
    case 1: return s.p * (v3 - v1) + s.q * (v4 - v0);
    case 2: return s.p * (v2 - v1) + s.q * (v3 - v0);
    case 3: return s.p * (v2 + v1) + s.q * (v3 + v0);
    default: return s.c[0] * v0 + s.c[1] * v1 + s.c[2] * v2 + s.c[3] * v3 + s.c[4] * v4;
  }
}

struct TileArgs {
  const double* b;
  double* x;
  Layout lay;
  int64_t tiles_per_outer, num_tiles;
  int Q;            // chunk heads per column (n / K)
  int G;            // cluster size
  int rows_per_cta; // n / G
  int stages;       // log2 Q
  int vc_slab;      // VC with nparts > 1 (two levels): slab row 0 is the GPU interface
  int l2_W;         // > 0: rows <= l2_W and >= n - l2_W of every slab stored evict-last (window)
  int mode;         // 0: complete cyclic solve (p = 1); 1: y_D = D_i^{-1} b_i + planes (p >= 2);
                    // 2: complete acyclic solve (p = 1)
  int rows_box;     // TMA box rows (<= 256)
  int pcr_uniform;  // 1: per-stage multipliers below (cyclic uniform head system); 0: tables
  double ualpha[kMaxUniformStages], ugamma[kMaxUniformStages], uinv;
  const double* pcr_alpha;  // [stages][Q]
  const double* pcr_gamma;  // [stages][Q]
  const double* pcr_inv;    // [Q]
  double* plane_yf;  // mode 1: y_D at interior row 1
  double* plane_yl;  // mode 1: y_D at row n-1
  double* plane_bt;  // mode 1: b at row 0 (b~_i)
  // fused compact-scheme RHS stencil (LAYOUT 2), see Stencil5
  Stencil5 st;
  const double* halo_lo;  // [2][m]: rows n-2, n-1 of the slab above
  const double* halo_hi;  // [2][m]: rows 0, 1 of the slab below
  int halo_wrap;          // one partition: halo rows are the slab's own wrap rows (TMA), no planes
  int halo_tma;           // nparts > 1: halo rows from the planes by TMA (xmap), not per-thread loads
  unsigned long long* trace;  // measurement only (CTRI_TILE_TRACE=<cta>)
  int trace_cta;              // the CTA whose tiles are stamped
  int trace_off;              // its first stamped tile (CTRI_TILE_TRACE_OFF)
  int vc_dbg;                 // experiment knob CTRI_VC_DBG, compiled in with -DCTRI_VC_EXPERIMENTS
                              // (bit 0: no window finalisation; bits 2, 3: finalisation without its
                              // stores / loads -- wrong results, timing only)
  // fused reduced phase (LAYOUT 3, nparts > 1): the window rows of every tile stay
  // in shared memory while the tile's (c = b~ - u y_D[1], y_D[n-1]) go to every rank's mailbox
  // as LL words; one tile later x~_i, x~_{i+1} = rows i, i+1 of A^{-1} applied to the gathered
  // b^ (reading R21), and the window rows are corrected (Eq. xi_app) and stored once.
  int f_P, f_row, f_W, f_srw, f_cyclic;  // reduced rows, this rank's row, window, stash rows/slot
  unsigned long long* f_peer[8];         // every rank's fused mailbox (own included)
  int64_t f_m;                           // plane length (batch columns)
  double f_g0[8], f_g1[8];               // rows f_row and f_row + 1 of A^{-1}
  const double *f_S, *f_R;               // slab-level S_i, R_i (n - 1)
  unsigned int *f_epoch, *f_done;        // device epoch of the solve, CTA completion count
  int* f_err;                            // deadline error word
  // virtual-partition chain (LAYOUT 4, nparts == 1 with vp > 1): one cluster solves the vp
  // partitions of a column group back to back, gathers their planes on chip (c_v = b~_v -
  // u y_v[first] in CTA 0, y_v[last] in CTA G-1, exchanged by st.async), solves the vp-row
  // reduced system per column with the plan's PCR multipliers (fold R3) and
  // finalises the window rows of every partition (Eq. xi_app, R15) while the next group is
  // being solved: they were stored with an L2 evict-last hint and are read back from L2, so
  // HBM sees 16 B per point.  f_S / f_R carry the slab-level S, R tables.
  int vc_vp, vc_W, vc_q, vc_cyclic;
  int64_t vc_groups;                     // column groups (num_tiles / vp)
  double vc_alpha[4 * 8], vc_gamma[4 * 8], vc_inv[8];  // [stage][row] PCR of the vp-row system
};

// on-chip pentadiagonal local solve (ptile.cu): kernel arguments and plan-time configuration
struct PTileArgs {
  double* x;
  Layout lay;                 // the (virtual) slabs as the kernel sees them
  int64_t tiles_per_outer, num_tiles;
  int Q, G, stages, mode;     // chunk heads per column, cluster, head-system PCR stages, mode
  const double* tab;          // [stages][Q][4] alpha | [stages][Q][4] gamma | [Q][4] fold
  double* planes4;            // mode 1: [4][pm] c0 | c1 | w0 | w1 per (virtual) slab column
  int64_t pm;
  unsigned long long* trace;  // measurement only (CTRI_TILE_TRACE): one CTA's phase stamps
  int trace_cta;
};
struct PTileConfig {
  bool ok = false;
  int G = 0, Q = 0, stages = 0, mode = 0, grid = 0, smem = 0;
  std::vector<double> tab, consts;  // head-system tables; chunk LU, S0, S1, R0, R1 (30 each)
  double* d_tab = nullptr;
};

struct TileConfig {
  bool ok = false;
  int variant = 0;  // index into the tile variant table (tile.cu)
  int C = 0, NT = 0, STAGES = 0, MINB = 0;  // columns per tile, threads, ring slots, CTAs/SM
  int SUB = 1;                              // sub-tiles per CTA tile (ring slot granularity)
  bool pcr_uniform = false;
  bool contig = false;                      // contiguous solve axis variant
  int K = 0, G = 0, Q = 0;
  int smem_bytes = 0;
  int grid = 0;  // CTAs launched (multiple of G)
  bool deriv_ok = false;               // fused-stencil instantiation configured
  int smem_deriv = 0, grid_deriv = 0;
  bool fused_ok = false;               // fused reduced-phase instantiation configured (LAYOUT 3)
  int smem_fused = 0, grid_fused = 0, fused_srw = 0;
  bool vc_ok = false;                  // virtual-partition chain instantiation (LAYOUT 4)
  int smem_vc = 0, grid_vc = 0;
  std::vector<double> consts;  // serialized TileConsts<K> (l, u, then 4 tables of K-1)
  PcrTables pcr;
  double* d_pcr = nullptr;     // device: alpha | gamma | inv
};

// ---- fused device-initiated reduced phase (p2p.cu) ----
constexpr int kMaxP2PRanks = 16;  // real multi-GPU: <= 8 per box; loopback tests up to 16
constexpr int kMaxP2PSteps = 16;
// %globaltimer stamps of the P2P kernels, per CTA: start, y sent, y received, after schedule
// step s (3 + s), x~ received, end
constexpr int kP2PTrace = 24, kTrStart = 0, kTrYSent = 1, kTrYRecv = 2, kTrStep0 = 3,
              kTrXRecv = 3 + kMaxP2PSteps, kTrEnd = 4 + kMaxP2PSteps;
constexpr int kMaxAG = 8;  // all-gather reduced solve (CTRI_FLAG_ALLGATHER): nparts <= 8
// One rank's part of a reduced-system schedule step (factor.h Schedule):
//   v <- w v - c0 u0 - c1 u1, u_k received in mailbox slot k from rank src_k;
//   this rank's pre-step v is sent to ranks dst_k, slot dslot_k.
struct P2PStep {
  double w, c0, c1;
  int8_t src0, src1, dst0, dst1, dslot0, dslot1;
};
struct P2PRank {
  int rank;
  double* x;
  const double *yf, *yl, *bt;
  double* xnext;                 // x~_{i+1} per batch column, read by the window pass
  const double* f;               // derivative halo kernel: this rank's f slab
  double *halo_lo, *halo_hi;     // derivative halo planes [2][m]
  unsigned long long* mbox;      // own mailbox of LL words (2 epoch copies)
  unsigned int* epoch;           // per slice: epoch of the last solve (device-resident, so a
                                 // solve captured in a CUDA graph advances it on every replay)
  unsigned long long* peer_mbox[kMaxP2PRanks];  // every rank's mailbox as addressable here
  P2PStep step[kMaxP2PSteps];
  double ag0[kMaxAG], ag1[kMaxAG];  // all-gather mode: rows i and i+1 of A^{-1} (zeros past p)
  const double* planes4;         // pentadiagonal: c0 | c1 | w0 | w1 of this row, plane k at k * pstride
  int64_t pstride;               // pentadiagonal: plane stride (m, or m * vp with virtual rows)
  const double* ainv;            // pentadiagonal all-gather: [2p][2p] reduced inverse
  const double* ppcr;            // pentadiagonal pairwise: this rank's [step][8] A0 | A1, fold [4]
};
struct P2PArgs {
  int p, q, cyclic, nslices, full;  // q = number of schedule steps
  int allgather;                    // 1: one all-gather round + A^{-1} rows instead of the schedule
  int pdl;                          // launched with programmatic stream serialization
  int64_t slice_cols, m, W;
  int64_t copy_words;               // mailbox words of one epoch copy of the reduced-phase region
  Layout lay;
  double l, u;
  const double *S, *R;
  int* err;
  unsigned long long deadline_ns;  // every LL wait gives up after this long (default 20 s)
  int test_drop_rank;              // TEST ONLY (CTRI_TEST_P2P_DROP_RANK): this reduced row never
                                   // sends its y plane, so its neighbour hits the deadline
  unsigned long long* trace;  // CTRI_FLAG_TIMING / CTRI_P2P_TRACE: [grid][kP2PTrace] stamps
  P2PRank rk[kMaxP2PRanks];
};
// nranks_launch > 1: cooperative (loopback); nrows: rows launched (ranks x virtual rows)
cudaError_t launch_reduced_p2p(const P2PArgs& A, int nranks_launch, cudaStream_t s, int nrows = 1);
int p2p_slices(int64_t m, int nranks_launch, int num_sms, int kind);  // 0 schedule, 1 all-gather,
                                                                       // 2 penta all-gather, 3 penta PCR
cudaError_t launch_reduced_allgather_r2(const P2PArgs& A, int nranks_launch, cudaStream_t s);
cudaError_t launch_reduced_penta_pcr(const P2PArgs& A, int nranks_launch, cudaStream_t s);
int64_t p2p_copy_words(int64_t m, int q, int p, bool allgather, int planes = 2);
size_t p2p_mailbox_words(int64_t copy_words, int64_t m, bool halo);
cudaError_t launch_halo_p2p(const P2PArgs& A, int nranks_launch, cudaStream_t s);

struct Plan {
  // configuration
  int64_t gdims[3] = {0, 0, 0};
  int sd = 0, p = 1, rank = 0, cyclic = 1;
  uint32_t flags = 0;
  Bands bands{};
  Layout lay;           // local slab
  int vp = 1;           // virtual partitions of the slab solved as separate partitions on this
                        // GPU (nparts == 1 only; the paper's method with more partitions than GPUs)
  Layout tlay;          // layout the local-solve kernels see: (outer*vp, n/vp, inner)
  int rvp = 1;          // rows per rank of the reduced system: vp ("virtual rows"), or 1 when the
                        // virtual partitions are chained inside the tile kernel (two levels)
  int device = 0;
  int num_sms = 0;
  bool loopback = false;

  // host tables
  Partition part;       // S_i, R_i, L^, D^, U^ of the reduced system's partitions (n/rvp rows)
  Partition vpart;      // the same for the local kernels' (virtual) partitions (n/vp rows)
  int64_t vwindow = 0;  // window rows per end at the virtual level
  PcrTables vpcr;       // two levels: acyclic vp-row system of the slab's internal interfaces
  PcrTables gpcr;       // GPU-level PCR over the p reduced rows (power-of-two or acyclic)
  Schedule sched;       // reduced-system step schedule (PCR / detach / fold / reattach)
  int64_t window = 0;   // rows per end for (a4)
  double inv_closure = 0;  // p = 1 generic path: 1/(L^ + D^ + U^)

  // device tables
  double* d_cp = nullptr;       // generic local solve Thomas factors (n-1)
  double* d_inv_den = nullptr;
  double* d_S = nullptr;        // S_i, R_i of the reduced system's partitions (n/rvp - 1)
  double* d_R = nullptr;
  double* d_vS = nullptr;       // two levels: S, R of the virtual partitions (n/vp - 1)
  double* d_vR = nullptr;

  // planes (m doubles each)
  double *yf = nullptr, *yl = nullptr, *bt = nullptr, *yl_prev = nullptr, *bh = nullptr,
         *recv_m = nullptr, *recv_p = nullptr, *xt = nullptr, *xt_next = nullptr;
  // derivative halos: [2][m] each
  double *halo_lo = nullptr, *halo_hi = nullptr, *send_lo = nullptr, *send_hi = nullptr;

  // local-solve kernel selection
  int local_kernel = 0;  // 0 generic, 1 tile (strided axis)
  TileConfig tile;

  // e2e staging (ctri_solve_host); with one partition and a large slab the copies and the
  // solve are pipelined over column chunks, each solved by a sub-plan of the chunk's shape
  double* d_stage_b = nullptr;
  double* d_stage_x = nullptr;
  Plan* e2e_sub = nullptr;
  int e2e_mode = -1;   // -1 undecided, 0 sequential, 1 chunks along outer, 2 chunks along inner
  int e2e_nch = 0;
  cudaStream_t e2e_h2d = nullptr, e2e_d2h = nullptr;
  std::vector<cudaEvent_t> e2e_ev;  // [start, end, h2d[nch], solved[nch]]

  // fused P2P reduced phase
  bool p2p = false;
  bool allgather = false;         // CTRI_FLAG_ALLGATHER: reduced system by A^{-1} rows
  std::vector<double> ainv;       // [p][p] A^{-1} (all-gather mode)
  int p2p_nslices = 0;
  bool fused = false;                  // (a2)-(a4) fused into the tile kernel (LAYOUT 3)
  bool vchain = false;                 // nparts == 1, vp > 1: (a2)-(a4) inside the tile kernel
                                       // (LAYOUT 4, no k_reduced_local / k_window launches)
  double fg0[8] = {0}, fg1[8] = {0};   // fused: rows rank, rank + 1 of A^{-1}
  unsigned int* d_fctr = nullptr;      // fused: [epoch, CTA completion count]
  int64_t p2p_off = 0;                 // words before the P2P-kernel region of the mailbox
  int64_t p2p_vrow_words = 0;          // mailbox words per virtual row (both epoch copies)
  void* mbox_alloc = nullptr;          // own LL mailbox (cudaMalloc, IPC-exported)
  unsigned int* d_epoch = nullptr;     // per-slice solve epochs of the fused P2P kernel
  size_t mbox_bytes = 0;
  std::vector<void*> peer_alloc;       // peer allocations as mapped here (IPC) or direct
  std::vector<bool> peer_ipc;          // opened with cudaIpcOpenMemHandle
  unsigned long long deadline_ns = 20ull * 1000000000ull;  // P2P wait deadline (CTRI_TEST_P2P_DEADLINE_MS)
  int test_drop_rank = -1;             // CTRI_TEST_P2P_DROP_RANK (tests of the deadline path)
  int* d_err = nullptr;                // device view of the error word (p2p deadline)
  int* h_err = nullptr;                // the same word in mapped pinned host memory: the host
                                       // reads it without a sync and poisons the plan
  unsigned int* d_hepoch = nullptr;    // per-slice epochs of the derivative halo exchange
  int64_t halo_off = 0;                // words before the halo region of the mailbox
  unsigned long long* d_trace = nullptr;  // P2P per-round stamps (CTRI_FLAG_TIMING / CTRI_P2P_TRACE)
  int trace_ctas = 0;
  unsigned long long epoch = 0;

  // comm
  ncclComm_t comm = nullptr;
  std::vector<Plan*> group;  // loopback peers (index = rank)

  // pentadiagonal plan (r = 2, penta.cu)
  int r = 1;                      // interface rows per partition: 1 tridiagonal, 2 pentadiagonal
  double bands5[5] = {0, 0, 0, 0, 0};
  Penta pt;
  double pcinv[4] = {0, 0, 0, 0};  // p == 1: inverse of the 2x2 closure
  double *d_plu = nullptr;         // [4][N]: lam1 | lam2 | nu1 | inv_mu
  double *d_pSR = nullptr;         // [4][N]: S0 | S1 | R0 | R1
  double *d_ainv = nullptr;        // [2p][2p] reduced inverse (p > 1)
  double *d_planes4 = nullptr;     // [4][m]: c0 | c1 | w0 | w1  (c = b~ - U~ y_i, w = L~ y_i)
  double *d_xnext2 = nullptr;      // [2][m]: x~_{i+1}
  PTileConfig ptc;                 // on-chip local solve (local_kernel 4)
  PentaPcr vppcr;                  // nparts == 1, vp > 1: 2x2-block PCR over the vp partitions
  double *d_vppcr = nullptr;       // [stages][vp][4] alpha | gamma, [vp][4] fold
  bool ppcr = false;               // pairwise 2x2-block PCR reduced solve (else all-gather)
  bool pdense = false;             // one GPU, cyclic, vp not a power of two: d_vppcr holds A^-1
  int ppcr_steps = 0;
  double *d_ppcr = nullptr;        // this rank's [step][8] A0 | A1 and fold [4]
  std::vector<P2PStep> pstep;      // this rank's partners per block-PCR step
  int64_t p2p_copy = 0;            // mailbox words per epoch copy (pentadiagonal plans)

  // stats
  uint64_t solves = 0;
  std::vector<cudaEvent_t> ev;  // timing events
  bool timed_valid = false;
  int launches_per_solve = 0;
};

// Measurement / experiment knobs read once per process (the per-solve launch path must not
// scan the environment): CTRI_NO_PDL, CTRI_P2P_TRACE, CTRI_TILE_TRACE, CTRI_TILE_COPY_ONLY.
inline bool env_knob(const char* name) { return std::getenv(name) != nullptr; }
inline bool knob_no_pdl() { static const bool v = env_knob("CTRI_NO_PDL"); return v; }
inline bool knob_p2p_trace() { static const bool v = env_knob("CTRI_P2P_TRACE"); return v; }
inline bool knob_tile_trace() { static const bool v = env_knob("CTRI_TILE_TRACE"); return v; }
inline bool knob_copy_only() { static const bool v = env_knob("CTRI_TILE_COPY_ONLY"); return v; }
// CTRI_NO_VCHAIN: virtual partitions finish with k_reduced_local + k_window (A/B measurement;
// read at plan creation, not on the solve path)
inline bool knob_no_vchain() { return env_knob("CTRI_NO_VCHAIN"); }
// CTRI_TWO_LEVEL: nparts > 1 with virtual partitions chained in the tile kernel (plan creation)
inline bool knob_two_level() { return env_knob("CTRI_TWO_LEVEL"); }

// kernels.cu launchers (return cudaError_t of the launch)
cudaError_t launch_local_generic(const Plan& P, const double* b, double* x, cudaStream_t s);
cudaError_t launch_bhat(const Plan& P, cudaStream_t s);
cudaError_t launch_pcr_stage(const Plan& P, int k, bool last, cudaStream_t s);
cudaError_t launch_backsub(const Plan& P, double* x, cudaStream_t s);
cudaError_t launch_reduced_local(const Plan& P, double* x, cudaStream_t s);
cudaError_t launch_window(const Plan& P, double* x, const double* next, cudaStream_t s);
// penta.cu (r = 2)
ctri_status penta_plan_tables(Plan* P, cudaStream_t s, std::string* why);
cudaError_t launch_penta_local(const Plan& P, const double* b, double* x, cudaStream_t s);
cudaError_t launch_penta_window(const Plan& P, double* x, cudaStream_t s);
cudaError_t launch_penta_reduced_local(const Plan& P, double* x, cudaStream_t s);
bool ptile_configure(Plan& P, std::string* why);
cudaError_t launch_ptile(const Plan& P, const double* b, double* x, cudaStream_t s);
// CTRI_PENTA_COLUMN_SERIAL: pentadiagonal plans keep the column-serial local solve (A/B)
inline bool knob_penta_serial() { return env_knob("CTRI_PENTA_COLUMN_SERIAL"); }
cudaError_t launch_pack_halo(const Plan& P, const double* f, cudaStream_t s);
cudaError_t launch_stencil(const Plan& P, const double* f, double* rhs, const Stencil5& st,
                           cudaStream_t s);
bool tile_configure(Plan& P, std::string* why);
const char* tile_variant_name(int v);
cudaError_t launch_tile(const Plan& P, const double* b, double* x, cudaStream_t s,
                        const Stencil5* st = nullptr);

}  // namespace ctri
