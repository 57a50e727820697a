// tile.cu -- the hot kernel: cluster-tile local solve of (a1) for a strided solve axis.
//
// PAPER.md P:317 solves D_i y_i = b_i "on the shared memory" by generalized PCR; here the
// same partition method (Eqs. system1/system2, xi, Li_hat..bi_hat, xi_app) is
// applied hierarchically ON CHIP (R16):
//   * a column of the slab (n rows, fixed batch index) is cut into Q = n/K chunks of K rows;
//     the first row of each chunk is its head (the chunk-level interface unknown, like x~_i),
//     the other K-1 rows its interior;
//   * each thread holds one chunk of one column in registers and eliminates the interior
//     with plan-time Thomas factors (the register leaf: y_c = D_K^{-1} b_c, Eq. yi);
//   * the Q heads of a column form a tridiagonal system with RHS b^_c = b~_c - l y_{c-1}[last]
//     - u y_c[first] (Eq. bi_hat) and plan-time coefficients (Eqs. Li_hat..Ui_hat at chunk
//     level), solved by PCR in shared memory of the CTA owning that column; the Q
//     chunks of a column live in the G CTAs of a thread-block cluster and reach the owner
//     through distributed shared memory;
//   * each chunk is back-substituted, x_c = y_c - S_K x~_c - R_K x~_{c+1} (Eq. xi_app), and
//     stored.
// The batch is streamed in column tiles of C columns: TMA (cp.async.bulk.tensor) moves tile
// t+STAGES into a shared-memory ring while tile t is computed from registers, so HBM sees
// one read of b and one write of x: 16 B per grid point.
//
// mode 0: nparts = 1 cyclic (complete solve; the head system is cyclic)
// mode 1: nparts > 1: y_D = D_i^{-1} b_i on rows 1..n-1 (row 0 is the GPU interface, decoupled
//         as a dummy head), plus the planes y_D[1], y_D[n-1], b[0] for (a2)
// mode 2: nparts = 1 acyclic (complete solve)
// mode 3: measurement only (CTRI_TILE_COPY_ONLY): x = b through the same TMA ring and stores
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "internal.h"
#include "ptx.cuh"

namespace ctri {

// CTRI_VC_DBG experiment bits of the virtual-partition chain (timing studies only: they break
// results) are compiled in only with -DCTRI_VC_EXPERIMENTS
#ifdef CTRI_VC_EXPERIMENTS
constexpr bool kVcExperiments = true;
#else
constexpr bool kVcExperiments = false;
#endif

template <int K, int C, int NT, int SUB, int SLOTS, int MINB, int LAYOUT>
__global__ void __launch_bounds__(NT, MINB)
    k_tile(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap hmap,
           const __grid_constant__ CUtensorMap xmap, const TileArgs A, const TileConsts<K> T) {
  // LAYOUT 0: strided solve axis; 1: contiguous solve axis; 2: strided + fused compact-derivative
  // RHS stencil (a0): the kernel reads f, forms b in registers and never writes it
  // LAYOUT 3: strided + fused reduced phase (nparts > 1): window rows stashed in shared memory,
  // planes to every rank's mailbox as LL words, finalised one tile later (TileArgs f_*)
  constexpr bool CONTIG = (LAYOUT == 1);
  constexpr bool DERIV = (LAYOUT == 2);
  constexpr bool FUSED = (LAYOUT == 3);
  // LAYOUT 4: nparts == 1 with vp virtual partitions: the cluster walks the vp partitions of a
  // column group back to back and finishes (a2)-(a4) on chip (TileArgs vc_*)
  constexpr bool VC = (LAYOUT == 4 || LAYOUT == 5);
  constexpr bool VC_SLAB = (LAYOUT == 5);  // two levels (nparts > 1): slab row 0 is the GPU interface
  constexpr int HALO = DERIV ? 2 : 0;     // stencil half-width (rows)
  static_assert(K >= 4 && NT % C == 0 && (C == 4 || C == 8 || C == 16 || C == 32 || C == 64), "tile geometry");
  static_assert(!CONTIG || (NT / C == 32 && SUB == 1 && SLOTS == 1), "contiguous: 32 chunks/CTA");
  static_assert(!DERIV || SUB == 1, "fused stencil: whole-tile ring slots");
  static_assert(!VC || (SUB == 1 && !CONTIG), "virtual-partition chain: strided whole tiles");
  static_assert(SLOTS >= SUB, "ring must hold one tile");
  constexpr int CPC = NT / C;             // chunks per CTA
  constexpr int ROWS = CPC * K;           // rows per CTA
  // strided axis: rows of C columns (C*8 bytes) share the 32 banks with PRD-1 other rows;
  // contiguous axis: chunks are (K+2)*8 bytes apart, half-warps rotate by one row
  constexpr int PRD = CONTIG ? 2 : (C >= 16 ? 1 : 16 / C);
  constexpr int CSTRIDE = K + 2;          // contiguous axis: padded chunk stride (doubles)
  // TMA ring: SLOTS slots of one sub-tile each (SUB sub-tiles of SR rows per CTA tile), so up to
  // SLOTS sub-tiles are in flight while the current tile is computed from registers
  constexpr int CPS = CPC / SUB;          // chunks per sub-tile
  constexpr int SR = CPS * K;             // rows per sub-tile
  constexpr int RING = CONTIG ? C * CPC * CSTRIDE : (SR + 2 * HALO) * C;  // doubles per slot
  static_assert(K % PRD == 0, "K must be a multiple of the bank period");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int Q = A.Q;
  const int stages = A.stages;
  double* ring = reinterpret_cast<double*>(smem_raw);
  double* ex_bt = ring + (size_t)SLOTS * RING;        // owner: b~ of every head it owns
  double* ex_yf = ex_bt + NT;                        // owner: y_c[first]
  double* ex_yl = ex_yf + NT;                        // owner: y_c[last]
  double* pb0 = ex_yl + NT;                          // owner: PCR ping-pong
  double* pb1 = pb0 + NT;
  double* rx_a = pb1 + NT;                           // holder: x~_c of its chunk
  double* rx_b = rx_a + NT;                          // holder: x~_{c+1}
  double* s_alpha = rx_b + NT;                       // PCR multipliers [stages][Q]
  double* s_gamma = s_alpha + (size_t)stages * Q;
  double* s_inv = s_gamma + (size_t)stages * Q;      // [Q]
  const bool tab = !A.pcr_uniform;  // per-row PCR multipliers in smem (acyclic head systems)
  uint64_t* mbar = reinterpret_cast<uint64_t*>(tab ? s_inv + Q : s_alpha);  // [SLOTS] ring, ex, rx
  uint64_t* mbar_ex = mbar + SLOTS;
  uint64_t* mbar_rx = mbar_ex + 1;
  uint64_t* mbar_red = mbar_rx + 1;  // VC: [2] planes of a column group's owned columns
  // FUSED: [2][f_srw][C] window rows (128-byte aligned: TMA-store source)
  // (offset arithmetic on smem_raw, not on an integer address: the compiler must keep seeing
  // a shared-memory pointer, or every stash access becomes a generic LD/ST)
  double* f_stash = reinterpret_cast<double*>(
      smem_raw + ((reinterpret_cast<unsigned char*>(mbar_red + 2) - smem_raw + 127) & ~(ptrdiff_t)127));
  double* f_red = FUSED ? f_stash + (size_t)2 * A.f_srw * C : nullptr;  // [2][NT] partial x~
  double* f_sr = FUSED ? f_red + 2 * NT : nullptr;  // [2][f_srw]: S, R of the stashed rows
  // VC (per owned column, C/G of them): [2 groups][8] c_v and y_v[last] planes, [2 groups][9]
  // x~ (row vp: x~ past the last partition); [2][2W+1] S, R of the window rows in block order
  // (rows 0..W, then nv-W..nv-1)
  const int vc_cpo = C / A.G;  // owned columns per CTA
  double* vc_c = f_stash;
  double* vc_yl = vc_c + 2 * 8 * vc_cpo;
  double* vc_xt = vc_yl + 2 * 8 * vc_cpo;
  double* vc_sr = vc_xt + 2 * 9 * vc_cpo;
  double* vc_pcr = vc_sr + 2 * (VC ? 2 * A.vc_W + 1 : 0);  // [72] PCR multipliers, vp-row system
  // [4 groups][2]: outer index and column tile of the last column groups (written once per
  // group by thread 0, so no thread divides on the tile path)
  int* vc_gtab = reinterpret_cast<int*>(vc_pcr + 72);
  // [2][kVcFin][NT] pairs of window values in flight (16-byte cp.async, double-buffered)
  double* vc_buf = reinterpret_cast<double*>(
      smem_raw + ((reinterpret_cast<unsigned char*>(vc_gtab + 8) - smem_raw + 15) & ~(ptrdiff_t)15));
  double** vc_bptr = reinterpret_cast<double**>(vc_buf + 8 * NT);  // [2][NT]: the blocks in flight

  const int tid = threadIdx.x;
  // strided axis: lanes run over the C columns of a tile row (coalesced rows);
  // contiguous axis: lanes run over the 32 chunks of one column, warps over columns
  const int j = CONTIG ? tid / 32 : tid % C;   // column within the tile
  const int cl = CONTIG ? tid % 32 : tid / C;  // chunk within this CTA
  const int G = A.G;
  const uint32_t g = (G > 1) ? dev::cluster_ctarank() : 0u;
  const int c = (int)g * CPC + cl;  // chunk index within the column (0..Q-1)
  const int cpo = C / G;            // columns owned per CTA
  const uint32_t owner = (uint32_t)(j / cpo);
  const int slot = (j % cpo) * Q + c;
  const int oj = tid / Q, oc = tid - (tid / Q) * Q;  // reduced row owned by this thread
  const int prev_row = oj * Q + ((oc - 1) & (Q - 1));
  const int ocol = (int)g * cpo + oj;                // tile column of the owned row
  // rotation of the smem row reads so that the PRD groups of a warp hit disjoint banks
  const int rot = CONTIG ? ((tid & 31) >> 4) : ((tid & 31) / C) % PRD;

  if (tab) {
    for (int i = tid; i < stages * Q; i += NT) {
      s_alpha[i] = A.pcr_alpha[i];
      s_gamma[i] = A.pcr_gamma[i];
    }
    for (int i = tid; i < Q; i += NT) s_inv[i] = A.pcr_inv[i];
  }
  if (tid < SLOTS) dev::mbar_init(dev::smem_u32(mbar + tid), 1);
  if (tid == SLOTS) dev::mbar_init(dev::smem_u32(mbar_ex), 1);
  if (tid == SLOTS + 1) dev::mbar_init(dev::smem_u32(mbar_rx), 1);
  if (VC && tid == SLOTS + 2) dev::mbar_init(dev::smem_u32(mbar_red), 1);
  if (VC && tid == SLOTS + 3) dev::mbar_init(dev::smem_u32(mbar_red + 1), 1);
  if (VC) {  // S, R of the window rows (Eq. xi_app, R15) by block row ri: slab row ri (ri <= W),
             // else nv - 2W - 1 + ri; row 0 is x~ itself
    const int W = A.vc_W, R2 = 2 * W + 1;
    const int64_t nv = A.lay.n;
    for (int ri = tid; ri < R2; ri += NT) {
      const int64_t r = ri <= W ? ri : nv - R2 + ri;
      vc_sr[ri] = r >= 1 ? A.f_S[r - 1] : 0.0;
      vc_sr[R2 + ri] = r >= 1 ? A.f_R[r - 1] : 0.0;
    }
    for (int i = tid; i < 72; i += NT)
      vc_pcr[i] = i < 32 ? A.vc_alpha[i] : i < 64 ? A.vc_gamma[i - 32] : i < 72 ? A.vc_inv[i - 64] : 0.0;
  }
  if (tid == 0) dev::fence_mbar_init();
  __syncthreads();
  if (G > 1) dev::cluster_sync();  // barriers initialised cluster-wide before any st.async

  const uint32_t ncl = (G > 1) ? dev::ncluster_x() : gridDim.x;
  const int64_t first = (G > 1) ? (int64_t)dev::cluster_id_x() : (int64_t)blockIdx.x;
  // tile of this cluster's iteration itx (-1 past the end)
  auto tile_at = [&](int64_t itx) -> int64_t {
    const int64_t t = first + itx * (int64_t)ncl;
    return t < A.num_tiles ? t : -1;
  };
  // VC: the cluster walks column groups first, first + ncl, ...; within a group the vp
  // partitions one after the other (tile (og * vp + v, ct)); positions advance incrementally,
  // one 64-bit division per group
  // (32-bit: the host checks that column groups and tiles per outer index fit)
  const int vcp = VC ? A.vc_vp : 1;
  const int vtpo = (int)A.tiles_per_outer;
  auto vc_og = [&](int gi) { return ((int)first + gi * (int)ncl) / vtpo; };  // outer index of group gi
  auto vc_ct = [&](int gi) {                                                   // its column tile
    const int cg = (int)first + gi * (int)ncl;
    return cg - (cg / vtpo) * vtpo;
  };
  auto vc_has = [&](int gi) { return (int64_t)first + (int64_t)gi * ncl < A.vc_groups; };
  int vq = 0, vgi = 0;              // partition within the group, groups completed
  constexpr uint32_t kSubBytes = (uint32_t)(SR + 2 * HALO) * C * (uint32_t)sizeof(double);
  const int boxr = A.rows_box;
  const int row0 = (int)g * ROWS;
  const uint64_t pol = dev::policy_evict_first();

  // sub-tile sequence number seq -> (tile first + (seq / SUB) * ncl, part seq % SUB), slot seq % SLOTS
  // (VC: the caller passes the tile's outer index and first column, o_vc >= 0)
  auto issue = [&](int64_t seq, int64_t o_vc = -1, int64_t col_vc = 0) {
    int o, col0;
    if (VC) {
      if (o_vc < 0) return;
      o = (int)o_vc;
      col0 = (int)col_vc;
    } else {
      const int64_t t = tile_at(seq / SUB);
      if (t < 0) return;
      o = (int)(t / A.tiles_per_outer);
      col0 = (int)(t - (int64_t)o * A.tiles_per_outer) * C;
    }
    const int h = (int)(seq % SUB);
    const int s = (int)(seq % SLOTS);
    const uint32_t bar = dev::smem_u32(mbar + s);
    double* dst = ring + (size_t)s * RING;
    const int r0 = row0 + h * SR;
    dev::fence_proxy_async();
    dev::mbar_expect_tx(bar, kSubBytes);
    for (int r = 0; r < SR; r += boxr)
      dev::tma_load_3d(dev::smem_u32(dst + (size_t)(r + HALO) * C), &tmap, col0, r0 + r, o, bar, pol);
    if (DERIV) {  // stencil halo rows row0-2, row0-1 and row0+ROWS, +1: zero-filled outside the
                  // slab (and then taken from the halo planes), or with one partition the
                  // periodic wrap rows n-2, n-1 / 0, 1 of the same column tile
      // (nparts > 1: the slab-edge CTAs take them from the halo planes, [2][2][m], through
      // xmap: rows 0, 1 the slab above, rows 2, 3 the slab below)
      const int lo = (A.halo_wrap && g == 0) ? (int)A.lay.n - HALO : row0 - HALO;
      const int hi = (A.halo_wrap && (int)g == G - 1) ? 0 : row0 + ROWS;
      const uint32_t dlo = dev::smem_u32(dst), dhi = dev::smem_u32(dst + (size_t)(ROWS + HALO) * C);
      if (A.halo_tma && g == 0) dev::tma_load_3d(dlo, &xmap, col0, o, 0, bar, pol);
      else dev::tma_load_3d(dlo, &hmap, col0, lo, o, bar, pol);
      if (A.halo_tma && (int)g == G - 1) dev::tma_load_3d(dhi, &xmap, col0, o, 2, bar, pol);
      else dev::tma_load_3d(dhi, &hmap, col0, hi, o, bar, pol);
    }
  };
  const int hsub = cl / CPS, lc = cl - (cl / CPS) * CPS;  // my sub-tile and chunk within it

  // remote addresses: my (b~, y_first, y_last) -> owner; my x~ -> holders of chunks oc, oc-1
  // (mapped where they are used: mapa is one instruction, a live address a register)
  auto rmap = [&](const void* p, uint32_t rank) {
    const uint32_t a = dev::smem_u32(p);
    return G > 1 ? dev::mapa(a, rank) : a;
  };
  // holder thread of (column ocol, chunk cc): strided tid = cl*C + j, contiguous tid = j*32 + cl
  auto holder_tid = [&](int cc) { return CONTIG ? ocol * 32 + (cc % CPC) : (cc % CPC) * C + ocol; };
  const int ocm = (oc - 1) & (Q - 1);  // chunk oc's holder gets x~_oc as x_a, chunk oc-1's as x_b

  // contiguous axis: ONE TMA load per tile through a 3-D view (row in chunk, chunk, column) of
  // the slab with a box of K+2 rows per chunk: the 2 rows past each chunk are out of bounds of
  // the view and arrive zero-filled, so the ring gets the padded (K+2)-double chunk stride that
  // keeps the lane-per-chunk reads conflict-free -- no per-thread copies
  auto issue_contig = [&](int64_t t) {
    if (tid != 0) return;
    const uint32_t bar = dev::smem_u32(mbar);
    dev::fence_proxy_async();
    dev::mbar_expect_tx(bar, (uint32_t)(C * CPC * CSTRIDE) * 8u);
    dev::tma_load_3d(dev::smem_u32(ring), &tmap, 0, (int)(g * CPC), (int)(t * C), bar, pol);
  };
  if (CONTIG) {
    if (first < A.num_tiles) issue_contig(first);
  } else if (tid == 0) {
    if (VC) issue(0, vc_has(0) ? (int64_t)vc_og(0) * vcp : -1, (int64_t)vc_ct(0) * C);
    else
      for (int s = 0; s < SLOTS; ++s) issue(s);
  }

  // measurement only (CTRI_TILE_TRACE): CTA 0 stamps its first 64 tiles' phases
  unsigned long long* tr = (A.trace && (int)blockIdx.x == A.trace_cta) ? A.trace : nullptr;
  auto stamp = [&](int it_, int k) {  // tiles trace_off .. trace_off + 63
    if (tr && tid == 0 && it_ >= A.trace_off && it_ < A.trace_off + 64) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      tr[(it_ - A.trace_off) * 16 + k] = tt;
    }
  };
  int it = 0;
  // ---- fused reduced phase (FUSED): roles, epoch, finalisation of a previous tile ----
  const bool f_top = FUSED && g == 0;
  const bool f_bot = FUSED && (int)g == G - 1;
  const int64_t f_n = A.lay.n;
  const int f_W = FUSED ? A.f_W : 0;
  const int f_bbase = (G == 1) ? f_W + 1 : 0;  // stash row of slab row n - W - 1
  const int64_t f_b0 = f_n - f_W - 1;           // first stashed row of the bottom block
  // rows k in [f_kb, f_ke) of this thread's chunk are stashed, at stash row k + f_soff (a chunk
  // never holds both window blocks: tile_configure requires n >= 2(W+1) + K)
  int f_kb = K, f_ke = 0, f_soff = 0;
  if (FUSED) {
    const int64_t rc0 = (int64_t)c * K;
    if (f_top && rc0 <= f_W) {
      f_kb = 0;
      f_ke = (int)std::min<int64_t>(K, f_W + 1 - rc0);
      f_soff = (int)rc0;
    } else if (f_bot && rc0 + K > f_b0) {
      f_kb = (int)std::max<int64_t>(0, f_b0 - rc0);
      f_ke = K;
      f_soff = f_bbase + (int)(rc0 - f_b0);
    }
  }
  uint32_t f_ep = 0;
  unsigned long long f_deadline = 0;
  if (FUSED) {
    f_ep = *reinterpret_cast<volatile unsigned int*>(A.f_epoch) + 1u;
    f_deadline = dev::globaltimer_ns() + 20ull * 1000000000ull;
    // slab-level S, R of the rows this CTA stashes (stash row index -> slab row)
    for (int i = tid; i < A.f_srw; i += NT) {
      int64_t r = -1;
      if (f_top && i <= f_W) r = i;
      else if (f_bot && i >= f_bbase && i <= f_bbase + f_W) r = f_b0 + (i - f_bbase);
      f_sr[i] = (r >= 1) ? A.f_S[r - 1] : 0.0;
      f_sr[A.f_srw + i] = (r >= 1) ? A.f_R[r - 1] : 0.0;
    }
    __syncthreads();
  }
  // plane q, reduced row r, column jo of the current epoch copy (LL words: 2 per value)
  auto f_word = [&](int q, int r, int64_t jo) -> int64_t {
    return 2 * (((int64_t)(f_ep & 1u) * 2 * A.f_P + (int64_t)q * A.f_P + r) * A.f_m + jo);
  };
  unsigned long long f_w[4] = {0, 0, 0, 0};  // prefetched LL words of the tile to finalise
  auto f_prefetch = [&](int64_t tp) {
    const int64_t op = tp / A.tiles_per_outer;
    const int64_t cj = (tp - op * A.tiles_per_outer) * C + (tid % C);
    const int kg = tid / C;
    if (cj < A.lay.inner && kg < A.f_P) {
      const int64_t jo = op * A.lay.inner + cj;
      const unsigned long long* mb = A.f_peer[A.f_row];
      dev::ll_load(mb + f_word(0, kg, jo), &f_w[0], &f_w[1]);
      if (A.f_cyclic || kg > 0) dev::ll_load(mb + f_word(1, (kg + A.f_P - 1) % A.f_P, jo), &f_w[2], &f_w[3]);
    }
  };
  // x~_i, x~_{i+1} of tile tp for every column, then Eq. xi_app on its stashed window rows
  auto f_finalize = [&](int64_t tp, int slotp) {
    stamp(it, 8);
    if (tid == 0) dev::bulk_wait_read_all();  // the previous TMA store has read its stash slot
    const int64_t op = tp / A.tiles_per_outer;
    const int64_t colp = (tp - op * A.tiles_per_outer) * C;
    const int kg = tid / C;
    const int64_t cj = colp + (tid % C);
    double a0 = 0.0, a1 = 0.0;
    if (cj < A.lay.inner && kg < A.f_P) {
      const int64_t jo = op * A.lay.inner + cj;
      const unsigned long long* mb = A.f_peer[A.f_row];
      double ck = 0.0, ylp = 0.0;
      bool ok = true;
      if (dev::ll_ready(f_w[0], f_w[1], f_ep)) ck = dev::ll_value(f_w[0], f_w[1]);
      else ok = dev::ll_wait(mb + f_word(0, kg, jo), f_ep, f_deadline, &ck);
      const bool lft = A.f_cyclic || kg > 0;
      if (lft && ok) {
        if (dev::ll_ready(f_w[2], f_w[3], f_ep)) ylp = dev::ll_value(f_w[2], f_w[3]);
        else ok = dev::ll_wait(mb + f_word(1, (kg + A.f_P - 1) % A.f_P, jo), f_ep, f_deadline, &ylp);
      }
      if (!ok) *reinterpret_cast<volatile int*>(A.f_err) = 1;
      const double bh = ck - (lft ? T.l * ylp : 0.0);  // Eq. bi_hat
      a0 = A.f_g0[kg] * bh;
      a1 = A.f_g1[kg] * bh;
    }
    stamp(it, 9);
    f_red[tid] = a0;
    f_red[NT + tid] = a1;
    __syncthreads();
    stamp(it, 10);
    double* f_x = f_red;  // [2][C] x~_i, x~_{i+1} per column (f_red's first 2C are read first)
    double xa_j = 0.0, xb_j = 0.0;
    if (tid < C) {
#pragma unroll
      for (int q = 0; q < NT / C; ++q) {  // fixed order: deterministic
        xa_j += f_red[q * C + tid];
        xb_j += f_red[NT + q * C + tid];
      }
    }
    __syncthreads();
    if (tid < C) {
      f_x[tid] = xa_j;
      f_x[C + tid] = xb_j;
    }
    __syncthreads();
    {  // Eq. xi_app on the stashed window rows (R15), spread over all threads; row 0 is x~_i
      double* __restrict__ stp = f_stash + (size_t)slotp * A.f_srw * C;
      const double* __restrict__ sS = f_sr;
      const double* __restrict__ sR = f_sr + A.f_srw;
      const double* __restrict__ fx = f_x;
      for (int e = tid; e < A.f_srw * C; e += NT) {
        const int si = e / C, jj = e - (e / C) * C;
        const bool used = (f_top && si <= f_W) || (f_bot && si >= f_bbase && si <= f_bbase + f_W);
        if (!used) continue;
        const double xa = fx[jj], xb = fx[C + jj];
        stp[e] = (f_top && si == 0) ? xa : stp[e] - sS[si] * xa - sR[si] * xb;
      }
    }
    stamp(it, 12);
    dev::fence_proxy_async();  // generic-proxy smem writes -> visible to the TMA store
    stamp(it, 13);
    __syncthreads();
    stamp(it, 14);
    if (tid == 0) {  // the corrected window blocks go out through TMA (off the LSU store path)
      const uint32_t sb = dev::smem_u32(f_stash + (size_t)slotp * A.f_srw * C);
      if (f_top) dev::tma_store_3d(&xmap, sb, (int)colp, 0, (int)op);
      if (f_bot) dev::tma_store_3d(&xmap, sb + (uint32_t)(f_bbase * C * 8), (int)colp, (int)f_b0, (int)op);
      dev::bulk_commit();
    }
    stamp(it, 11);
  };

  // ---- virtual-partition chain (VC): roles, window rows, reduced solve, finalisation ----
  // Every CTA finishes the columns whose head systems it owns (cpo of them): it receives their
  // planes, solves their vp-row systems and finalises their window rows.  The window rows were
  // stored by the holder threads of those columns, whose later st.async head stores complete on
  // this CTA's exchange barrier with release semantics at cluster scope; the exchange wait is an
  // acquire at cluster scope, so those stores are visible here (no fence on the tile path).
  const int vc_W = VC ? A.vc_W : 0;
  const int vc_nv = VC ? (int)A.lay.n : 0;
  const int vc_R2 = 2 * vc_W + 1;  // window block rows per partition
  // rows k <= vc_wt of this thread's chunk are top-window rows (CTA 0), rows k >= vc_wb bottom
  // (CTA G-1): stored with an L2 evict-last hint, finalised one column group later
  const int vc_wt = (VC && g == 0) ? vc_W - c * K : -1;
  const int vc_wb = (VC && (int)g == G - 1) ? vc_nv - vc_W - c * K : K + 1;
  // (a2)-(a3) for the owned columns of group parity par: lane group of vp threads per column
  // (thread tid < cpo*vp: row v = tid % vp of column tid / vp): b^_v = c_v - l y_{v-1}[last]
  // (Eq. bi_hat), PCR over the vp rows by register shuffles with the plan's multipliers
  // (both partners may coincide, fold R3), x~_v = b^_v inv_v -> vc_xt[par][v]
  // (row vp: x~ right of the last partition, the wrap x~_0 or 0 when acyclic)
  auto vc_solve = [&](int par) {
    const int v = tid % vcp, jl = tid / vcp;
    const bool act = jl < cpo;
    const int vl = v == 0 ? vcp - 1 : v - 1;
    double bh = 0.0;
    if (act && !(VC_SLAB && v == 0)) {  // two levels: row 0 (the GPU interface) is decoupled
      const double ylp = (v > 0 || A.vc_cyclic) ? vc_yl[(par * 8 + vl) * cpo + jl] : 0.0;
      bh = vc_c[(par * 8 + v) * cpo + jl] - T.l * ylp;
    }
    for (int k = 0; k < A.vc_q; ++k) {
      const int sh = 1 << k;
      const double vm = __shfl_sync(0xffffffffu, bh, (v - sh) & (vcp - 1), vcp);
      const double vq = __shfl_sync(0xffffffffu, bh, (v + sh) & (vcp - 1), vcp);
      bh = bh - vc_pcr[k * 8 + v] * vm - vc_pcr[32 + k * 8 + v] * vq;
    }
    if (act) {
      const double xv = bh * vc_pcr[64 + v];
      vc_xt[(par * 9 + v) * cpo + jl] = xv;
      if (v == 0) vc_xt[(par * 9 + vcp) * cpo + jl] = A.vc_cyclic ? xv : 0.0;
    }
  };
  const bool vc_solver = VC && (tid / 32) < (cpo * vcp + 31) / 32;  // whole warps (shuffles)
  // window element i of this thread: block row tid / (cpo/2) + i * (NT / (cpo/2)), the pair of
  // owned columns 2 (tid % (cpo/2)) and the next: 16-byte copies, loads and stores
  constexpr int kVcFin = 2;  // host: (2W + 1) * C / G / 2 <= 2 NT
  const int vc_hp = cpo / 2;
  const int vc_jl = 2 * (tid % vc_hp);
  const int vc_r0 = tid / vc_hp, vc_rs = NT / vc_hp;
  auto gt_og = [&](int gi) { return vc_gtab[2 * (gi & 3)]; };
  auto gt_ct = [&](int gi) { return vc_gtab[2 * (gi & 3) + 1]; };
  auto vc_block = [&](int gi, int q) -> double* {  // (row 0, this thread's column pair) of a block
    const int64_t colp = (int64_t)gt_ct(gi) * C + (int64_t)g * cpo + vc_jl;
    if (colp >= A.lay.inner) return nullptr;  // (inner is even: the pair is whole or absent)
    return A.x + ((int64_t)(gt_og(gi) * vcp + q) * vc_nv) * A.lay.inner + colp;
  };
  auto vc_row = [&](int ri) { return ri <= vc_W ? ri : vc_nv - vc_R2 + ri; };
  // this thread's window rows as element offsets (host: nv * inner < 2^31)
  int vc_off[kVcFin];
#pragma unroll
  for (int i = 0; i < kVcFin; ++i) {
    const int ri = vc_r0 + i * vc_rs;
    vc_off[i] = ri < vc_R2 ? vc_row(ri) * (int)A.lay.inner : 0;
  }
  // y of the window rows (stored >= vp tiles earlier by the holder CTAs) -> this thread's
  // vc_buf slots by cp.async (L2 only), so nothing is held in registers meanwhile
  auto vc_load = [&](const double* blk, int bf) {
    if (blk) {
      double* bb = vc_buf + bf * kVcFin * 2 * NT;
#pragma unroll
      for (int i = 0; i < kVcFin; ++i) {
        const int ri = vc_r0 + i * vc_rs;
        if (ri < vc_R2 && ri != 0 && !(kVcExperiments && (A.vc_dbg & 8)))
          dev::cp_async_16(dev::smem_u32(bb + 2 * (i * NT + tid)), blk + vc_off[i]);
      }
    }
    dev::cp_async_commit();
  };
  // Eq. xi_app on the loaded window rows (row 0 of the partition := x~_q), stored once
  // (two levels: slab row 0 keeps its role as the GPU interface -- not written here -- and the
  // finalised rows 1 and n-1 of the slab, y_D[first] and y_D[last], go to the planes of the
  // reduced system across the GPUs)
  auto vc_store = [&](double* blk, int gp, int q, int bf) {
    if (!blk) return;
    const double* bb = vc_buf + bf * kVcFin * 2 * NT;
    const double* xt = vc_xt + (gp & 1) * 9 * cpo;
    const double2 xa = *reinterpret_cast<const double2*>(xt + q * cpo + vc_jl);
    const double2 xb = *reinterpret_cast<const double2*>(xt + (q + 1) * cpo + vc_jl);
#pragma unroll
    for (int i = 0; i < kVcFin; ++i) {
      const int ri = vc_r0 + i * vc_rs;
      if (ri >= vc_R2) break;
      const double s = vc_sr[ri], r = vc_sr[vc_R2 + ri];
      const double2 y = *reinterpret_cast<const double2*>(bb + 2 * (i * NT + tid));
      const double x0 = ri == 0 ? xa.x : y.x - s * xa.x - r * xb.x;
      const double x1 = ri == 0 ? xa.y : y.y - s * xa.y - r * xb.y;
      if (VC_SLAB) {
        if (q == 0 && ri == 0) continue;
        const int64_t pj = (int64_t)gt_og(gp) * A.lay.inner + (int64_t)gt_ct(gp) * C + (int64_t)g * cpo + vc_jl;
        if (q == 0 && ri == 1) { A.plane_yf[pj] = x0; A.plane_yf[pj + 1] = x1; }
        if (q == vcp - 1 && ri == vc_R2 - 1) { A.plane_yl[pj] = x0; A.plane_yl[pj + 1] = x1; }
      }
      if (!(kVcExperiments && (A.vc_dbg & 4))) dev::st_global_cs_v2(blk + vc_off[i], x0, x1);
    }
  };
  // the window block finalised at tile itx: that of tile itx - vp - 1 (partition q - 1 of the
  // previous group, or the last partition of the group before it); false if none
  auto vc_target = [&](int gi, int q, int* fg, int* fq) -> bool {
    *fq = q >= 1 ? q - 1 : vcp - 1;
    *fg = q >= 1 ? gi - 1 : gi - 2;
    return *fg >= 0 && !(kVcExperiments && (A.vc_dbg & 1));
  };

  for (;; ++it) {
    int64_t t;
    int vog = 0, vct = 0;  // VC: this group's outer index and column tile (after the barrier)
    if (VC) {
      if (!vc_has(vgi)) break;
      if (tid == 0 && vq == 0) {  // a new column group: its position into the table
        vc_gtab[2 * (vgi & 3)] = vc_og(vgi);
        vc_gtab[2 * (vgi & 3) + 1] = vc_ct(vgi);
      }
      t = 0;  // (VC addresses the tile through vog, vct)
    } else {
      t = tile_at(it);
      if (t < 0) break;
    }
    stamp(it, 0);
    const int vc_q = vq;                            // VC: partition of this tile
    const int vc_gi = vgi;                          // VC: column group (this cluster's count)
    if (FUSED && (f_top || f_bot) && it > 0) f_prefetch(t - ncl);
    const int64_t seq = (int64_t)it * SUB + hsub;
    const int s = (int)(seq % SLOTS);
    if (tid == 0 && A.mode != 3) {  // arm this tile's exchange barriers (remote bytes may race ahead)
      dev::mbar_expect_tx(dev::smem_u32(mbar_ex), (uint32_t)NT * 3u * 8u);
      dev::mbar_expect_tx(dev::smem_u32(mbar_rx), (uint32_t)NT * 2u * 8u);
      if (VC && vc_q == 0)  // c_v and y_v[last] of this group's owned columns
        dev::mbar_expect_tx(dev::smem_u32(mbar_red + (vc_gi & 1)), (uint32_t)(2 * vcp * cpo * 8));
    }
    dev::mbar_wait(dev::smem_u32(mbar + s), (uint32_t)(seq / SLOTS) & 1u);
    double* tile = ring + (size_t)s * RING;
    if (DERIV && !A.halo_wrap && !A.halo_tma) {
      // slab-edge CTAs: the halo rows outside the slab come from the neighbour slabs (halo planes)
      const int64_t oo = t / A.tiles_per_outer;
      const int64_t cc0 = (t - oo * A.tiles_per_outer) * C;
      if (g == 0 && tid < HALO * C) {
        const int64_t cc = cc0 + (tid % C);
        if (cc < A.lay.inner) tile[(tid / C) * C + tid % C] = A.halo_lo[(tid / C) * A.lay.m() + oo * A.lay.inner + cc];
      }
      if ((int)g == G - 1 && tid < HALO * C) {
        const int64_t cc = cc0 + (tid % C);
        if (cc < A.lay.inner)
          tile[(ROWS + HALO + tid / C) * C + tid % C] = A.halo_hi[(tid / C) * A.lay.m() + oo * A.lay.inner + cc];
      }
      __syncthreads();
    }
    double v[K + 2 * HALO];
#pragma unroll
    for (int k = 0; k < K + 2 * HALO; k += PRD) {
      double a[PRD];
#pragma unroll
      for (int i = 0; i < PRD; ++i) {
        const int kk = k + ((i + rot) % PRD);
        a[i] = CONTIG ? tile[(j * CPC + cl) * CSTRIDE + kk] : tile[(lc * K + kk) * C + j];
      }
#pragma unroll
      for (int m = 0; m < PRD; ++m) {  // a[i] holds row k + (i + rot) % PRD
        double r = a[0];
#pragma unroll
        for (int i = 1; i < PRD; ++i)
          if ((i + rot) % PRD == m) r = a[i];
        v[k + m] = r;
      }
    }
    if (DERIV) {  // b_k = sum_j c_j f_{k+j} (compact-scheme RHS, Stencil5), in place;
                  // one uniform branch per tile selects the scheme's pair form
      const double p = A.st.p, q = A.st.q;
      switch (A.st.kind) {
        case 1:
#pragma unroll
          for (int k = 0; k < K; ++k) v[k] = p * (v[k + 3] - v[k + 1]) + q * (v[k + 4] - v[k]);
          break;
        case 2:
#pragma unroll
          for (int k = 0; k < K; ++k) v[k] = p * (v[k + 2] - v[k + 1]) + q * (v[k + 3] - v[k]);
          break;
        case 3:
#pragma unroll
          for (int k = 0; k < K; ++k) v[k] = p * (v[k + 2] + v[k + 1]) + q * (v[k + 3] + v[k]);
          break;
        default:
#pragma unroll
          for (int k = 0; k < K; ++k)
            v[k] = A.st.c[0] * v[k] + A.st.c[1] * v[k + 1] + A.st.c[2] * v[k + 2] +
                   A.st.c[3] * v[k + 3] + A.st.c[4] * v[k + 4];
      }
    }
    stamp(it, 1);
    __syncthreads();  // every thread has its chunk in registers: stage s is free
    if (CONTIG) {
      if (t + ncl < A.num_tiles) issue_contig(t + ncl);
    } else if (tid == 0) {
      if (VC) {  // the next tile: next partition of this group, or partition 0 of the next group
        if (vq + 1 < vcp) issue(it + 1, (int64_t)gt_og(vgi) * vcp + vq + 1, (int64_t)gt_ct(vgi) * C);
        else issue(it + 1, vc_has(vgi + 1) ? (int64_t)vc_og(vgi + 1) * vcp : -1, (int64_t)vc_ct(vgi + 1) * C);
      } else {
        for (int hh = 0; hh < SUB; ++hh) issue((int64_t)it * SUB + hh + SLOTS);  // freed slots
      }
    }
    if (VC) {
      vog = gt_og(vgi);
      vct = gt_ct(vgi);
    }
    // global column: strided axis (o, col) with col < inner; contiguous axis column = o
    const int64_t o = CONTIG ? t * C + j : (VC ? (int64_t)vog * vcp + vq : t / A.tiles_per_outer);
    const int64_t col = CONTIG ? 0 : (VC ? (int64_t)vct * C : (t - o * A.tiles_per_outer) * C) + j;
    const bool valid = CONTIG ? (o < A.lay.outer) : (col < A.lay.inner);
    auto store_chunk = [&]() {
      if (!valid) return;
      double* xp = A.x + (o * A.lay.n + (int64_t)c * K) * A.lay.inner + col;
      if (VC && (vc_wt >= 0 || vc_wb <= K)) {  // a chunk holding window rows (warp-uniform:
        // the chunk is the warp): its y stays in L2 until the finaliser reads the window rows
        // back (the whole chunk: no per-row test on the store path); row 0 of the partition is
        // left to the finaliser (x~)
        const uint64_t pol_last = dev::policy_evict_last();
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (c != 0 || k != 0) dev::st_global_hint(xp + (int64_t)k * A.lay.inner, v[k], pol_last);
        return;
      }
      if (FUSED) {  // window rows wait in shared memory for x~ (finalised one tile later)
        double* stp = f_stash + (size_t)(it & 1) * A.f_srw * C + (size_t)f_soff * C + j;
#pragma unroll
        for (int k = 0; k < K; ++k) {
          if (k >= f_kb && k < f_ke) stp[k * C] = v[k];
          else dev::st_global_cs(xp + (int64_t)k * A.lay.inner, v[k]);
        }
        return;
      }
      if (CONTIG) {
#pragma unroll
        for (int k = 0; k < K; k += 4) dev::st_global_cs_v4(xp + k, v[k], v[k + 1], v[k + 2], v[k + 3]);
      } else if ((LAYOUT == 0 || LAYOUT == 2) && A.l2_W > 0 &&
                 ((g == 0 && c * K <= A.l2_W) || ((int)g == G - 1 && (c + 1) * K > (int)A.lay.n - A.l2_W))) {
        // nparts > 1, window rows of the whole solve fit in L2: the chunks holding them (whole
        // warps) store every row evict-last, so the window pass after the reduced phase reads
        // them from L2 instead of HBM
        const uint64_t pol_last = dev::policy_evict_last();
#pragma unroll
        for (int k = 0; k < K; ++k) dev::st_global_hint(xp + (int64_t)k * A.lay.inner, v[k], pol_last);
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) dev::st_global_cs(xp + (int64_t)k * A.lay.inner, v[k]);
      }
    };
    if (A.mode == 3) {  // measurement only: the same load/store pipeline without the solve
      store_chunk();
      continue;
    }

    // ---- chunk interior solve (rows 1..K-1), Thomas with plan-time factors (Eq. yi) ----
    const double btv = v[0];
    {
      double gg = v[1] * T.inv_den[0];
      v[1] = gg;
#pragma unroll
      for (int k = 2; k < K; ++k) {
        gg = fma(T.mlid[k - 1], gg, v[k] * T.inv_den[k - 1]);  // (v_k - l g_{k-1}) / den_k
        v[k] = gg;
      }
#pragma unroll
      for (int k = K - 2; k >= 1; --k) v[k] = fma(-T.cp[k - 1], v[k + 1], v[k]);
    }
    stamp(it, 2);
    // ---- (b~_c, y_c[first], y_c[last]) -> owner CTA, completing on its exchange barrier ----
    {
      const uint32_t bar = rmap(mbar_ex, owner);
      dev::st_async_f64(rmap(ex_bt + slot, owner), btv, bar);
      dev::st_async_f64(rmap(ex_yf + slot, owner), v[1], bar);
      dev::st_async_f64(rmap(ex_yl + slot, owner), v[K - 1], bar);
    }
    if (VC) {  // in the shadow of the exchange: (a2)-(a4) work of earlier tiles
      // x~ of the previous group's owned columns (its planes left at least a tile ago)
      if (vc_q == 0 && vc_gi > 0 && vc_solver) {
        const int par = (vc_gi - 1) & 1;
        dev::mbar_wait(dev::smem_u32(mbar_red + par), (uint32_t)(((vc_gi - 1) >> 1) & 1));
        vc_solve(par);
      }
      // start loading the next tile's target (stored >= vp tiles ago and acquired since); it
      // is finalised in the x~ shadow of the next tile, so the loads have a whole tile to land
      // (issued after this tile's stores they queued behind them: 0.5 us waits per tile)
      int fg, fq;
      stamp(it, 12);
      const int nq = vc_q + 1 < vcp ? vc_q + 1 : 0, ngi = vc_q + 1 < vcp ? vc_gi : vc_gi + 1;
      if (vc_target(ngi, nq, &fg, &fq)) {
        double* blk = vc_block(fg, fq);
        vc_bptr[((it + 1) & 1) * NT + tid] = blk;  // (this thread's own slot)
        vc_load(blk, (it + 1) & 1);
      } else {
        dev::cp_async_commit();  // (an empty group keeps the group count per tile)
      }
      stamp(it, 7);
    }
    // ---- owner: head system b^_c (Eq. bi_hat at chunk level), then PCR stages ----
    {
      // VC: an acquire at cluster scope once per column group suffices -- the window rows read
      // at tile it were stored at tile it - vp - 1 and released by the holders' head stores
      // of every later tile, and a group's first tile lies within the last vp tiles (the
      // acquire also invalidates L1: CCTL.IVALL in SASS, so not on every tile)
      if (VC && vq == 0) dev::mbar_wait_acq_cluster(dev::smem_u32(mbar_ex), (uint32_t)it & 1u);
      else dev::mbar_wait(dev::smem_u32(mbar_ex), (uint32_t)it & 1u);
      stamp(it, 3);
      const double lt = (A.mode == 2 && oc == 0) ? 0.0 : T.l * ex_yl[prev_row];  // acyclic top
      double bh = ex_bt[tid] - lt - T.u * ex_yf[tid];
      if (A.mode == 1 && oc == 0) bh = 0.0;  // slab row 0 is the GPU interface, not in D_i
      if (Q <= 32) {
        // the Q heads of an owned column are Q consecutive lanes of one warp (oc = lane % Q):
        // every PCR stage is a pair of register shuffles, no shared memory and no block barrier
        for (int k = 0; k < stages; ++k) {
          const int sh = 1 << k;
          const double vm = __shfl_sync(0xffffffffu, bh, (oc - sh) & (Q - 1), Q);
          const double vp = __shfl_sync(0xffffffffu, bh, (oc + sh) & (Q - 1), Q);
          const double al = tab ? s_alpha[k * Q + oc] : A.ualpha[k];
          const double ga = tab ? s_gamma[k * Q + oc] : A.ugamma[k];
          bh = bh - al * vm - ga * vp;
        }
      } else {
        double* cur = pb0;
        double* nxt = pb1;
        for (int k = 0; k < stages; ++k) {
          cur[tid] = bh;
          __syncthreads();
          const int sh = 1 << k;
          const double vm = cur[oj * Q + ((oc - sh) & (Q - 1))];
          const double vp = cur[oj * Q + ((oc + sh) & (Q - 1))];
          const double al = tab ? s_alpha[k * Q + oc] : A.ualpha[k];
          const double ga = tab ? s_gamma[k * Q + oc] : A.ugamma[k];
          bh = bh - al * vm - ga * vp;
          double* tmp = cur;
          cur = nxt;
          nxt = tmp;
        }
      }
      const double xt = bh * (tab ? s_inv[oc] : A.uinv);
      stamp(it, 4);
      // x~_oc -> x_a of chunk oc's holder and x_b of chunk oc-1's holder
      dev::st_async_f64(rmap(rx_a + holder_tid(oc), (uint32_t)(oc / CPC)), xt,
                        rmap(mbar_rx, (uint32_t)(oc / CPC)));
      dev::st_async_f64(rmap(rx_b + holder_tid(ocm), (uint32_t)(ocm / CPC)), xt,
                        rmap(mbar_rx, (uint32_t)(ocm / CPC)));
    }
    if (VC) {  // in the shadow of the x~ return: finalise this tile's target (loaded a tile ago;
               // the group just issued for the next tile may stay in flight)
      int fg, fq;
      stamp(it, 14);
      dev::cp_async_wait_group<1>();
      if (vc_target(vc_gi, vc_q, &fg, &fq)) vc_store(vc_bptr[(it & 1) * NT + tid], fg, fq, it & 1);
      stamp(it, 13);
    }
    dev::mbar_wait(dev::smem_u32(mbar_rx), (uint32_t)it & 1u);
    stamp(it, 5);
    const double xa = rx_a[tid];
    const double xb = (A.mode != 0 && c == Q - 1) ? 0.0 : rx_b[tid];  // x~_{i+1} outside D_i / acyclic end
    // ---- chunk back-substitution, Eq. xi_app at chunk level ----
    v[0] = (A.mode == 1 && c == 0) ? btv : xa;  // mode 1: slab row 0 keeps b~ (scratch)
#pragma unroll
    for (int k = 1; k < K; ++k) v[k] = v[k] - T.S[k - 1] * xa - T.R[k - 1] * xb;
    // FUSED: finalise the previous tile here, a whole tile after its stores were issued, so
    // the TMA store of its window rows does not queue behind them
    if (FUSED && (f_top || f_bot) && it > 0) f_finalize(t - ncl, (it - 1) & 1);
    store_chunk();
    stamp(it, 6);
    if (VC) {  // (a2) planes of partition vc_q -> the column's owner CTA: c_v (chunk 0) and
               // y_v[last] (chunk Q-1)
      const int par = (int)(vc_gi & 1);
      const int e = (par * 8 + vc_q) * cpo + (j % cpo);
      if (c == 0) {  // c_v = b~_v - u y_v[first]
        dev::st_async_f64(dev::mapa(dev::smem_u32(vc_c + e), owner), btv - T.u * v[1],
                          dev::mapa(dev::smem_u32(mbar_red + par), owner));
        if (VC_SLAB && vc_q == 0 && valid) A.plane_bt[(int64_t)vog * A.lay.inner + col] = btv;  // b~_i
      }
      if (c == Q - 1)
        dev::st_async_f64(dev::mapa(dev::smem_u32(vc_yl + e), owner), v[K - 1],
                          dev::mapa(dev::smem_u32(mbar_red + par), owner));
      if (++vq == vcp) {  // next column group
        vq = 0;
        ++vgi;
      }
    }
    if (valid && FUSED) {  // (a2) planes of this tile -> every rank's mailbox (all-gather, R21)
      const int64_t jo = o * A.lay.inner + col;
      if (c == 0) {
        const double cv = btv - T.u * v[1];  // c_i = b~_i - u y_i[first]
        for (int r = 0; r < A.f_P; ++r) dev::ll_store(A.f_peer[r] + f_word(0, A.f_row, jo), cv, f_ep);
      }
      if (c == Q - 1)
        for (int r = 0; r < A.f_P; ++r) dev::ll_store(A.f_peer[r] + f_word(1, A.f_row, jo), v[K - 1], f_ep);
    } else if (valid && !VC) {
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
  if (VC && vgi > 0) {  // finalise this cluster's last partitions
    const int gl = vgi - 1;
    dev::cluster_sync();  // the last tiles' window rows, stored by the holder CTAs, visible here
    dev::cp_async_wait_all();
    int fg, fq;
    if (vc_target(vgi, 0, &fg, &fq))  // loaded by the last tile (into buffer it & 1)
      vc_store(vc_bptr[(it & 1) * NT + tid], fg, fq, it & 1);
    if (vc_solver) {
      const int par = gl & 1;
      dev::mbar_wait(dev::smem_u32(mbar_red + par), (uint32_t)((gl >> 1) & 1));
      vc_solve(par);
    }
    __syncthreads();
    if (!(kVcExperiments && (A.vc_dbg & 1)))
      for (int q = 0; q < vcp; ++q) {
        double* blk = vc_block(gl, q);
        vc_load(blk, 0);
        dev::cp_async_wait_all();
        vc_store(blk, gl, q, 0);
      }
  }
  if (FUSED) {
    if ((f_top || f_bot) && it > 0) {  // the last tile of this cluster
      const int64_t tl = first + (int64_t)(it - 1) * ncl;
      f_prefetch(tl);
      f_finalize(tl, (it - 1) & 1);
    }
    if (tid == 0) dev::bulk_wait_all();  // TMA stores complete before the CTA's smem goes away
    __syncthreads();
    if (tid == 0) {  // the last CTA to finish publishes the epoch for the next solve
      const unsigned int prev = atomicAdd(A.f_done, 1u);
      if (prev == gridDim.x - 1) {
        *A.f_done = 0u;
        *A.f_epoch = f_ep;
      }
    }
  }
  if (G > 1) dev::cluster_sync();  // no CTA exits while peers may still address its smem
}

// ------------------------------------------------------------------------------------------
// variants: (C columns per tile, NT threads, STAGES smem ring depth, MINB CTAs per SM)
// ------------------------------------------------------------------------------------------
struct Variant {
  const char* name;
  int C, NT, SUB, SLOTS, MINB;
  bool contig;  // contiguous solve axis (inner == 1): cp.async into a padded ring
  int kmax = 32;  // largest rows-per-thread K
};
static const Variant kVariants[] = {
    {"c16t512s1", 16, 512, 1, 1, 1, false},
    {"c8t512s1", 8, 512, 1, 1, 1, false},
    {"c4t512s1", 4, 512, 1, 1, 1, false},
    {"c8t256s1", 8, 256, 1, 1, 2, false},
    {"c16t256s1", 16, 256, 1, 1, 2, false},
    {"c16t512s1_contig", 16, 512, 1, 1, 1, true},
    {"c8t256s1_contig", 8, 256, 1, 1, 2, true},
    {"c16t256x3", 16, 256, 2, 3, 2, false},   // half-tile ring slots, 1.5 tiles in flight
    {"c16t512x5", 16, 512, 4, 5, 1, false},   // quarter-tile ring slots, 1.25 tiles in flight
    {"c16t256x6", 16, 256, 4, 6, 2, false},   // quarter-tile slots, 1.5 tiles in flight
    {"c32t512s1", 32, 512, 1, 1, 1, false},   // 256-byte row segments
    {"c32t512x3", 32, 512, 2, 3, 1, false},   // 256-byte rows, half-tile ring slots
    {"c32t256x3", 32, 256, 2, 3, 2, false},   // 256-byte rows, 2 CTA/SM, half-tile slots
    {"c32t256s1", 32, 256, 1, 1, 2, false},   // 256-byte rows, 2 CTA/SM
    {"c32t256k16", 32, 256, 1, 1, 4, false, 16},  // 256-byte rows, K <= 16, 4 CTA/SM
    {"c16t256k16", 16, 256, 1, 1, 4, false, 16},  // 128-byte rows, K <= 16, 4 CTA/SM
    {"c32t256k16x3", 32, 256, 2, 3, 3, false, 16},  // K <= 16, half-tile slots, 3 CTA/SM
    {"c64t256s1", 64, 256, 1, 1, 2, false},   // 512-byte row segments, 4 chunks per CTA
    {"c64t512s1", 64, 512, 1, 1, 1, false},   // 512-byte row segments, 8 chunks per CTA
    {"c64t512x3", 64, 512, 2, 3, 1, false},   // 512-byte rows, half-tile ring slots
};
static constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

template <int K>
static void fill_consts(const TileConfig& tc, TileConsts<K>* T) {
  const double* c = tc.consts.data();
  T->l = c[0];
  T->u = c[1];
  const int n1 = K - 1;
  for (int k = 0; k < n1; ++k) {
    T->inv_den[k] = c[2 + k];
    T->mlid[k] = -c[0] * c[2 + k];
    T->cp[k] = c[2 + n1 + k];
    T->S[k] = c[2 + 2 * n1 + k];
    T->R[k] = c[2 + 3 * n1 + k];
  }
}

template <int K, int C, int NT, int SB, int S, int M, int LY>
static cudaError_t launch_one(const TileConfig& tc, const CUtensorMap& map, const CUtensorMap& hmap,
                              const CUtensorMap& xmap, const TileArgs& A, cudaStream_t s,
                              bool configure_only) {
  auto fn = k_tile<K, C, NT, SB, S, M, LY>;
  if (configure_only) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, tc.smem_bytes);
    return e;
  }
  TileConsts<K> T;
  fill_consts<K>(tc, &T);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(LY == 2 ? tc.grid_deriv : LY == 3 ? tc.grid_fused : LY >= 4 ? tc.grid_vc : tc.grid, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = LY == 2 ? tc.smem_deriv : LY == 3 ? tc.smem_fused : LY >= 4 ? tc.smem_vc : tc.smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = tc.G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, map, hmap, xmap, A, T);
}

template <int K, int C, int NT, int SB, int S, int M, int LY>
static const void* fn_ptr() {
  return reinterpret_cast<const void*>(&k_tile<K, C, NT, SB, S, M, LY>);
}

template <int C, int NT, int SB, int S, int M, int LY>
static cudaError_t dispatch_k(const TileConfig& tc, const CUtensorMap& map, const CUtensorMap& hmap,
                              const CUtensorMap& xmap, const TileArgs& A, cudaStream_t s, bool cfg_only,
                              const void** fp) {
  switch (tc.K) {
#define CTRI_K(KK)                                                       \
  case KK:                                                               \
    if (fp) *fp = fn_ptr<KK, C, NT, SB, S, M, LY>();                      \
    return fp ? cudaSuccess : launch_one<KK, C, NT, SB, S, M, LY>(tc, map, hmap, xmap, A, s, cfg_only);
    CTRI_K(4) CTRI_K(8) CTRI_K(16) CTRI_K(32)
#undef CTRI_K
  }
  return cudaErrorInvalidValue;
}

// kind 0: solve; 2: fused stencil + solve; 3: solve with the fused reduced phase (nparts > 1);
// 4: virtual-partition chain (nparts == 1, vp > 1)
static cudaError_t dispatch(const TileConfig& tc, int kind, const CUtensorMap& map,
                            const CUtensorMap& hmap, const CUtensorMap& xmap, const TileArgs& A,
                            cudaStream_t s, bool cfg_only, const void** fp = nullptr) {
#define CTRI_V(C, NT, SB, S, M, LY) return dispatch_k<C, NT, SB, S, M, LY>(tc, map, hmap, xmap, A, s, cfg_only, fp)
  if (kind == 4) {  // virtual-partition chain: strided whole-tile variants
    switch (tc.variant) {
      case 0: CTRI_V(16, 512, 1, 1, 1, 4);
      case 4: CTRI_V(16, 256, 1, 1, 2, 4);
      case 13: CTRI_V(32, 256, 1, 1, 2, 4);
      case 17: CTRI_V(64, 256, 1, 1, 2, 4);
      case 18: CTRI_V(64, 512, 1, 1, 1, 4);
    }
    return cudaErrorInvalidValue;
  }
  if (kind == 5) {  // the chain with two levels (nparts > 1, opt-in)
    switch (tc.variant) {
      case 4: CTRI_V(16, 256, 1, 1, 2, 5);
      case 13: CTRI_V(32, 256, 1, 1, 2, 5);
    }
    return cudaErrorInvalidValue;
  }
  if (kind == 3) {  // fused reduced phase: strided whole-tile variants
    switch (tc.variant) {
      case 0: CTRI_V(16, 512, 1, 1, 1, 3);
      case 4: CTRI_V(16, 256, 1, 1, 2, 3);
      case 13: CTRI_V(32, 256, 1, 1, 2, 3);
    }
    return cudaErrorInvalidValue;
  }
  if (kind == 2) {  // fused stencil: strided whole-tile variants with 16 or 32 columns
    switch (tc.variant) {
      case 0: CTRI_V(16, 512, 1, 1, 1, 2);
      case 4: CTRI_V(16, 256, 1, 1, 2, 2);
      case 13: CTRI_V(32, 256, 1, 1, 2, 2);
    }
    return cudaErrorInvalidValue;
  }
  switch (tc.variant) {
    case 0: CTRI_V(16, 512, 1, 1, 1, 0);
    case 1: CTRI_V(8, 512, 1, 1, 1, 0);
    case 2: CTRI_V(4, 512, 1, 1, 1, 0);
    case 3: CTRI_V(8, 256, 1, 1, 2, 0);
    case 4: CTRI_V(16, 256, 1, 1, 2, 0);
    case 5: CTRI_V(16, 512, 1, 1, 1, 1);
    case 6: CTRI_V(8, 256, 1, 1, 2, 1);
    case 7: CTRI_V(16, 256, 2, 3, 2, 0);
    case 8: CTRI_V(16, 512, 4, 5, 1, 0);
    case 9: CTRI_V(16, 256, 4, 6, 2, 0);
    case 10: CTRI_V(32, 512, 1, 1, 1, 0);
    case 11: CTRI_V(32, 512, 2, 3, 1, 0);
    case 12: CTRI_V(32, 256, 2, 3, 2, 0);
    case 13: CTRI_V(32, 256, 1, 1, 2, 0);
    case 14: CTRI_V(32, 256, 1, 1, 4, 0);
    case 15: CTRI_V(16, 256, 1, 1, 4, 0);
    case 16: CTRI_V(32, 256, 2, 3, 3, 0);
    case 17: CTRI_V(64, 256, 1, 1, 2, 0);
    case 18: CTRI_V(64, 512, 1, 1, 1, 0);
    case 19: CTRI_V(64, 512, 2, 3, 1, 0);
  }
#undef CTRI_V
  return cudaErrorInvalidValue;
}

// Preference order when CTRI_TILE_VARIANT is not set: the first variant whose geometry fits n.
// Measured on B200 (profiles/round1_tile_variants.md): 256-byte row segments with 2 CTA/SM
// first, then 128-byte tiles; portable clusters (<= 8) before 16-CTA ones.
static const int kPreference[] = {13, 4, 0, 12, 3, 1, 2, 6, 5};  // contiguous: c8t256 (2 CTA/SM) first

static int forced_variant() {
  const char* e = std::getenv("CTRI_TILE_VARIANT");  // experiment knob (bench sweeps)
  if (e)
    for (int v = 0; v < kNumVariants; ++v)
      if (!std::strcmp(e, kVariants[v].name)) return v;
  return -1;
}

const char* tile_variant_name(int v) { return (v >= 0 && v < kNumVariants) ? kVariants[v].name : "?"; }

static bool tile_configure_variant(Plan& P, int vi, std::string* why) {
  TileConfig& tc = P.tile;
  tc = TileConfig();
  const Layout& L = P.tlay;
  const Variant& V = kVariants[vi];
  if (V.contig) {
    if (L.inner != 1 || (L.n % 2) != 0) { *why = "contiguous variant needs inner == 1, n even"; return false; }
  } else if (L.inner < V.C || (L.inner % 2) != 0) {
    *why = "contiguous or narrow solve axis";
    return false;
  }
  if (L.outer > ((int64_t)1 << 30) || L.inner > ((int64_t)1 << 31) || L.n > ((int64_t)1 << 31)) {
    *why = "dims too large for TMA coordinates";
    return false;
  }
  const int cpc = V.NT / V.C;
  if (L.n % cpc != 0) { *why = "n not a multiple of chunks per CTA"; return false; }
  const int64_t kg = L.n / cpc;  // K * G
  int K = 0, G = 0;
  for (int k : {32, 16, 8, 4}) {
    if (k > V.kmax || kg % k) continue;
    const int64_t g = kg / k;
    if (g >= 1 && g <= kMaxClusterNonPortable && (g & (g - 1)) == 0 && V.C % g == 0) {
      K = k;
      G = (int)g;
      break;
    }
  }
  if (!K) { *why = "n not expressible as K*G*chunks (K<=32, G<=8)"; return false; }
  tc.variant = (int)(&V - kVariants);
  tc.contig = V.contig;
  tc.C = V.C;
  tc.NT = V.NT;
  tc.STAGES = V.SLOTS;
  tc.SUB = V.SUB;
  tc.MINB = V.MINB;
  const int Q = cpc * G;
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
  const bool cyc = (P.p == 1 && P.vp == 1 && P.cyclic);
  if (P.p > 1 || P.vp > 1) {  // dummy decoupled row 0 (the GPU interface), acyclic over the other heads
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
  const int rows_cta = cpc * K;
  if (cpc % V.SUB) { *why = "sub-tiles must split the chunks evenly"; return false; }
  // uniform (cyclic p = 1) head systems: the PCR multipliers are per-stage constants and travel
  // in the kernel parameters; otherwise per-row tables live in shared memory
  tc.pcr_uniform = tc.pcr.stages <= kMaxUniformStages;
  for (int k = 0; k < tc.pcr.stages && tc.pcr_uniform; ++k)
    for (int c = 1; c < Q; ++c)
      if (tc.pcr.alpha[(size_t)k * Q + c] != tc.pcr.alpha[(size_t)k * Q] ||
          tc.pcr.gamma[(size_t)k * Q + c] != tc.pcr.gamma[(size_t)k * Q])
        tc.pcr_uniform = false;
  for (int c = 1; c < Q && tc.pcr_uniform; ++c)
    if (tc.pcr.inv[c] != tc.pcr.inv[0]) tc.pcr_uniform = false;
  const size_t ring = V.contig ? (size_t)V.C * cpc * (K + 2) : (size_t)(rows_cta / V.SUB) * V.C;
  const size_t tables = tc.pcr_uniform ? 0 : (2 * (size_t)tc.pcr.stages + 1) * Q;
  tc.smem_bytes = (int)(sizeof(double) * ((size_t)V.SLOTS * ring + 7 * (size_t)V.NT + tables) +
                        8 * (V.SLOTS + 4));  // mbarriers: ring slots, ex, rx, red[2]
  // configure one instantiation (solve, or the fused-stencil one): smem attribute + grid
  auto setup = [&](int kind, int smem, int* grid_out) -> bool {
    const void* fn = nullptr;
    CUtensorMap dummy;
    TileArgs dA;
    dispatch(tc, kind, dummy, dummy, dummy, dA, 0, true, &fn);
    if (!fn || cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
      cudaGetLastError();
      *why = "cudaFuncSetAttribute(smem) failed";
      return false;
    }
    if (G > kMaxCluster &&
        cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      *why = "non-portable cluster size refused";
      return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G, 1, 1);
    cfg.blockDim = dim3(V.NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
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
    const int64_t num_tiles =
        V.contig ? (L.outer + V.C - 1) / V.C : L.outer * ((L.inner + V.C - 1) / V.C);
    *grid_out = (int)(std::min<int64_t>(nclusters, num_tiles) * G);
    return true;
  };
  if (!setup(0, tc.smem_bytes, &tc.grid)) return false;
  // fused-stencil instantiation (ctri_deriv): 4 extra ring rows per stage
  tc.deriv_ok = false;
  if (!V.contig && V.C >= 16 && V.SUB == 1 && (vi == 0 || vi == 4 || vi == 13) &&
      (P.flags & CTRI_FLAG_DERIV)) {
    tc.smem_deriv = tc.smem_bytes + (int)(sizeof(double) * 4 * V.C * V.SLOTS);
    std::string w2;
    std::swap(w2, *why);
    tc.deriv_ok = setup(2, tc.smem_deriv, &tc.grid_deriv);
    std::swap(w2, *why);
  }
  // fused reduced-phase instantiation (nparts > 1): a 2-slot stash of the window rows
  tc.fused_ok = false;
  if (!V.contig && V.SUB == 1 && (vi == 0 || vi == 4 || vi == 13) && P.p > 1 && P.vp == 1 &&
      P.window > 0) {
    const int64_t W = P.window;
    const int srw = (int)(G == 1 ? 2 * (W + 1) : W + 1);
    if (W + 1 <= 256 && ((G == 1 && 2 * (W + 1) + K <= L.n) || (G > 1 && W + 1 + K <= rows_cta))) {
      tc.fused_srw = srw;
      tc.smem_fused = tc.smem_bytes + 128 +
                      (int)(sizeof(double) * (2 * (size_t)srw * V.C + 2 * (size_t)V.NT + 2 * (size_t)srw));
      std::string w2;
      std::swap(w2, *why);
      tc.fused_ok = setup(3, tc.smem_fused, &tc.grid_fused);
      std::swap(w2, *why);
    }
  }
  // virtual-partition chain (nparts == 1, vp > 1): planes + x~ of two column groups and the
  // window-row S, R tables; the window blocks lie in the end CTAs (G >= 2) and fit the
  // finaliser's per-thread register budget (W + 1 <= 6 chunks per CTA)
  tc.vc_ok = false;
  if (!V.contig && V.SUB == 1 && (vi == 0 || vi == 4 || vi == 13 || vi == 17 || vi == 18) && P.vp > 1 &&
      (P.p == 1 || vi == 4 || vi == 13) &&
      P.vp <= 8 && G >= 2 && P.vwindow > 0 && !(P.flags & CTRI_FLAG_FULL_BACKSUB) &&
      !(P.flags & (CTRI_FLAG_NCCL_ROUNDS | CTRI_FLAG_ALLGATHER | CTRI_FLAG_FUSED_REDUCED)) &&
      (V.C / G) % 2 == 0 && (2 * P.vwindow + 1) * (V.C / G / 2) <= 2 * V.NT && P.vwindow + 1 <= rows_cta &&
      2 * P.vwindow + 1 < L.n &&
      L.outer * ((L.inner + V.C - 1) / V.C) < ((int64_t)1 << 31) &&  // 32-bit group arithmetic
      L.n * L.inner < ((int64_t)1 << 31)) {                           // 32-bit row offsets
    tc.smem_vc = tc.smem_bytes + 128 +
                 (int)(sizeof(double) * ((2 * 8 + 2 * 8 + 2 * 9) * (size_t)(V.C / G) + 2 * (2 * (size_t)P.vwindow + 1) +
                                         72 + 6 + 10 * (size_t)V.NT));  // vc_buf 8 NT, vc_bptr 2 NT
    std::string w2;
    std::swap(w2, *why);
    tc.vc_ok = setup(P.p > 1 ? 5 : 4, tc.smem_vc, &tc.grid_vc);
    std::swap(w2, *why);
  }
  tc.ok = true;
  return true;
}

bool tile_configure(Plan& P, std::string* why) {
  if (P.flags & CTRI_FLAG_GENERIC_LOCAL) { *why = "forced generic"; return false; }
  const int f = forced_variant();
  if (f >= 0) return tile_configure_variant(P, f, why);
  for (int pass = 0; pass < 2; ++pass)  // pass 0: portable clusters only
    for (int vi : kPreference)
      if (tile_configure_variant(P, vi, why) && (pass == 1 || P.tile.G <= kMaxCluster)) return true;
  return false;
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
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

cudaError_t launch_tile(const Plan& P, const double* b, double* x, cudaStream_t s,
                        const Stencil5* st) {
  const bool deriv = st != nullptr;
  const TileConfig& tc = P.tile;
  if (deriv && !tc.deriv_ok) return cudaErrorNotSupported;
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  const Layout& L = P.tlay;
  const int rows_cta = (tc.NT / tc.C) * tc.K;
  CUtensorMap map, hmap;
  std::memset(&map, 0, sizeof(map));
  std::memset(&hmap, 0, sizeof(hmap));
  if (tc.contig) {  // 3-D view (row in chunk, chunk, column), box K+2 rows: zero-padded chunks
    cuuint64_t gdim[3] = {(cuuint64_t)tc.K, (cuuint64_t)(L.n / tc.K), (cuuint64_t)L.outer};
    cuuint64_t gstride[2] = {(cuuint64_t)tc.K * 8, (cuuint64_t)L.n * 8};
    cuuint32_t box[3] = {(cuuint32_t)(tc.K + 2), (cuuint32_t)(tc.NT / tc.C), (cuuint32_t)tc.C};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(b), gdim, gstride,
                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  } else {
    cuuint64_t gdim[3] = {(cuuint64_t)L.inner, (cuuint64_t)L.n, (cuuint64_t)L.outer};
    cuuint64_t gstride[2] = {(cuuint64_t)L.inner * 8, (cuuint64_t)(L.n * L.inner * 8)};
    cuuint32_t box[3] = {(cuuint32_t)tc.C, (cuuint32_t)std::min(rows_cta / tc.SUB, 256), 1};
    cuuint32_t hbox[3] = {(cuuint32_t)tc.C, 2, 1};  // stencil halo rows (fused derivative)
    cuuint32_t estr[3] = {1, 1, 1};
    static const CUtensorMapL2promotion prom = [] {  // measurement knob, read once
      CUtensorMapL2promotion v = CU_TENSOR_MAP_L2_PROMOTION_NONE;
      if (const char* e = std::getenv("CTRI_TMA_L2_PROMOTION")) {
        if (!std::strcmp(e, "64")) v = CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
        if (!std::strcmp(e, "128")) v = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
        if (!std::strcmp(e, "256")) v = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
      }
      return v;
    }();
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(b), gdim,
                      gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, prom, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    if (deriv) {
      cr = enc(&hmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(b), gdim, gstride,
               hbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, prom,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
  }
  TileArgs A;
  A.b = b;
  A.x = x;
  A.lay = L;
  A.tiles_per_outer = tc.contig ? 1 : (L.inner + tc.C - 1) / tc.C;
  A.num_tiles = tc.contig ? (L.outer + tc.C - 1) / tc.C : L.outer * A.tiles_per_outer;
  A.Q = tc.Q;
  A.G = tc.G;
  A.rows_per_cta = rows_cta;
  A.rows_box = std::min(rows_cta / tc.SUB, 256);
  A.stages = tc.pcr.stages;
  A.mode = (P.p > 1 || P.vp > 1) ? 1 : (P.cyclic ? 0 : 2);
  if (knob_copy_only()) A.mode = 3;  // measurement knob: memory ceiling
  A.pcr_uniform = tc.pcr_uniform ? 1 : 0;
  for (int k = 0; k < kMaxUniformStages; ++k) {
    A.ualpha[k] = (tc.pcr_uniform && k < tc.pcr.stages) ? tc.pcr.alpha[(size_t)k * tc.Q] : 0.0;
    A.ugamma[k] = (tc.pcr_uniform && k < tc.pcr.stages) ? tc.pcr.gamma[(size_t)k * tc.Q] : 0.0;
  }
  A.uinv = tc.pcr.inv[0];
  A.trace = nullptr;
  A.trace_off = 0;
  if (knob_tile_trace()) {  // measurement only
    static unsigned long long* d_tr = nullptr;
    if (!d_tr) cudaMalloc(&d_tr, 64 * 16 * sizeof(unsigned long long));
    cudaMemsetAsync(d_tr, 0, 64 * 16 * sizeof(unsigned long long), s);
    A.trace = d_tr;
    A.trace_cta = std::atoi(std::getenv("CTRI_TILE_TRACE"));  // which CTA stamps (0 if not a number)
    const char* off = std::getenv("CTRI_TILE_TRACE_OFF");        // its first stamped tile
    A.trace_off = off ? std::atoi(off) : 0;
  }
  static const int vc_dbg = [] {  // experiment knob, read once per process
    const char* e = std::getenv("CTRI_VC_DBG");
    return e ? std::atoi(e) : 0;
  }();
  A.vc_dbg = vc_dbg;
  A.pcr_alpha = tc.d_pcr;
  A.pcr_gamma = tc.d_pcr + (size_t)tc.pcr.stages * tc.Q;
  A.pcr_inv = tc.d_pcr + (size_t)2 * tc.pcr.stages * tc.Q;
  A.plane_yf = P.yf;
  A.plane_yl = P.yl;
  A.plane_bt = P.bt;
  if (st) A.st = *st;
  // halo planes: rows n-2, n-1 of the slab above and rows 0, 1 of the slab below; with one
  // partition they are this slab's own rows (periodic wrap), packed into send_hi / send_lo
  A.halo_lo = (P.p == 1) ? P.send_hi : P.halo_lo;
  A.halo_hi = (P.p == 1) ? P.send_lo : P.halo_hi;
  // one partition: the periodic wrap rows come straight from the slab by TMA (no halo planes)
  A.halo_wrap = (P.p == 1) ? 1 : 0;
  const bool fused = !deriv && P.fused;
  const bool vchain = !deriv && P.vchain;
  // nparts > 1 without the chain: the window rows are stored with an L2 evict-last hint so the
  // window pass after the reduced phase finds them in L2 (all of them when they fit, the most
  // recent ones otherwise; the streaming rows are evict-first).  CTRI_L2_WINDOW_MB caps the
  // window bytes it is used for (default 64 MB: measured on 4 B200s, cfg3 0.0997 -> 0.0968 ms at
  // N = 4, while cfg5's 195 MB of window rows only slowed its tile kernel; 0 disables).
  A.l2_W = 0;
  static const int64_t l2_cap = [] {
    const char* e = std::getenv("CTRI_L2_WINDOW_MB");
    return (int64_t)(e ? std::atoi(e) : 64) << 20;
  }();
  if (P.p > 1 && !vchain && !fused && !tc.contig && P.window > 0 &&
      (2 * P.window + 1) * P.tlay.outer * P.lay.inner * 8 <= l2_cap)
    A.l2_W = (int)P.window;
  A.vc_slab = 0;
  if (vchain) {
    // nparts == 1: the vp-row system is the whole (cyclic or acyclic) reduced system (gpcr);
    // nparts > 1: the slab's internal interfaces, acyclic with the GPU interface decoupled
    // (vpcr), and the slab-level planes for the reduced system across GPUs
    const bool two = P.p > 1;
    const PcrTables& t = two ? P.vpcr : P.gpcr;
    A.vc_slab = two ? 1 : 0;
    A.vc_vp = P.vp;
    A.vc_W = (int)P.vwindow;
    A.vc_q = t.stages;
    A.vc_cyclic = two ? 0 : P.cyclic;
    A.vc_groups = A.num_tiles / P.vp;
    for (int i = 0; i < 32; ++i) A.vc_alpha[i] = A.vc_gamma[i] = 0.0;
    for (int k = 0; k < t.stages && k < 4; ++k)
      for (int v = 0; v < P.vp; ++v) {
        A.vc_alpha[k * 8 + v] = t.alpha[(size_t)k * P.vp + v];
        A.vc_gamma[k * 8 + v] = t.gamma[(size_t)k * P.vp + v];
      }
    for (int v = 0; v < 8; ++v) A.vc_inv[v] = v < P.vp ? t.inv[v] : 0.0;
    A.f_S = two ? P.d_vS : P.d_S;
    A.f_R = two ? P.d_vR : P.d_R;
  }
  if (fused) {
    A.f_P = P.p;
    A.f_row = P.rank;
    A.f_W = (int)P.window;
    A.f_srw = tc.fused_srw;
    A.f_cyclic = P.cyclic;
    for (int r = 0; r < 8; ++r) {
      A.f_peer[r] = (r < P.p) ? reinterpret_cast<unsigned long long*>(P.peer_alloc[r]) : nullptr;
      A.f_g0[r] = (r < P.p) ? P.fg0[r] : 0.0;
      A.f_g1[r] = (r < P.p) ? P.fg1[r] : 0.0;
    }
    A.f_m = P.lay.m();
    A.f_S = P.d_S;
    A.f_R = P.d_R;
    A.f_epoch = P.d_fctr;
    A.f_done = P.d_fctr + 1;
    A.f_err = P.d_err;
  }
  CUtensorMap xmap;
  std::memset(&xmap, 0, sizeof(xmap));
  A.halo_tma = 0;
  if (deriv && P.p > 1) {  // (A/B, 2 B200s: cfg5 0.554 -> 0.527 ms; per-thread loads remain for odd rows)
    // the halo planes as a (inner, outer, 4) tensor: box C x 1 x 2 = the two halo rows of a
    // column tile, landing in the ring as the tile's rows -2, -1 or ROWS, ROWS + 1
    cuuint64_t gdim[3] = {(cuuint64_t)P.lay.inner, (cuuint64_t)P.lay.outer, 4};
    cuuint64_t gstride[2] = {(cuuint64_t)P.lay.inner * 8, (cuuint64_t)(P.lay.m() * 8)};
    cuuint32_t box[3] = {(cuuint32_t)tc.C, 1, 2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, P.halo_lo, gdim, gstride, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr == CUDA_SUCCESS) A.halo_tma = 1;
  }
  if (fused) {  // output map for the TMA store of the finalised window blocks (W+1 rows)
    const Layout& L2 = P.tlay;
    cuuint64_t gdim[3] = {(cuuint64_t)L2.inner, (cuuint64_t)L2.n, (cuuint64_t)L2.outer};
    cuuint64_t gstride[2] = {(cuuint64_t)L2.inner * 8, (cuuint64_t)(L2.n * L2.inner * 8)};
    cuuint32_t box[3] = {(cuuint32_t)tc.C, (cuuint32_t)(P.window + 1), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, gdim, gstride, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  cudaError_t e = dispatch(tc, deriv ? 2 : (fused ? 3 : (vchain ? (P.p > 1 ? 5 : 4) : 0)), map, hmap, xmap, A, s, false);
  if (A.trace && e == cudaSuccess) {  // measurement only: print CTA 0's per-phase averages
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
    double fw[4] = {0, 0, 0, 0};
    int fcnt = 0;
    for (int i = 4; i < 60; ++i)  // fused finalisation: start, LL ready, reduced, stored
      if (h[i * 16 + 8] && h[i * 16 + 11]) {
        for (int k = 0; k < 3; ++k) fw[k] += (double)(h[i * 16 + 9 + k] - h[i * 16 + 8 + k]);
        ++fcnt;
      }
    double fz[3] = {0, 0, 0};
    for (int i = 4; i < 60; ++i)
      if (h[i * 16 + 10] && h[i * 16 + 14])
        for (int k = 0; k < 3; ++k) fz[k] += (double)(h[i * 16 + 12 + k] - h[i * 16 + 11 + k - (k == 0 ? 1 : 0)]);
    if (fcnt)
      std::fprintf(stderr, "[tile trace] fused finalise (ns): LL %.0f reduce %.0f correct+store %.0f "
                   "(correct %.0f fence %.0f sync %.0f)\n",
                   fw[0] / fcnt, fw[1] / fcnt, fw[2] / fcnt, fz[0] / fcnt, fz[1] / fcnt, fz[2] / fcnt);
    double vw[3] = {0, 0, 0};
    int vcnt = 0;
    for (int i = 4; i < 60; ++i)  // chain: exchange shadow (heads + solver, next loads), x~ shadow
      if (h[i * 16 + 12] && h[i * 16 + 7] && h[i * 16 + 13] && h[i * 16 + 14]) {
        vw[0] += (double)(h[i * 16 + 12] - h[i * 16 + 2]);
        vw[1] += (double)(h[i * 16 + 7] - h[i * 16 + 12]);
        vw[2] += (double)(h[i * 16 + 13] - h[i * 16 + 14]);
        ++vcnt;
      }
    if (vcnt)
      std::fprintf(stderr, "[tile trace] chain (ns): heads+solver %.0f next-block loads %.0f (exchange shadow); "
                   "wait+finalise %.0f (x~ shadow)\n", vw[0] / vcnt, vw[1] / vcnt, vw[2] / vcnt);
    if (cnt)
      std::fprintf(stderr,
                   "[tile trace] per tile (ns): ring_wait+lds %.0f thomas %.0f ex_wait %.0f pcr %.0f "
                   "rx_wait %.0f backsub+store %.0f loop %.0f total %.0f (%d tiles)\n",
                   acc[1] / cnt, acc[2] / cnt, acc[3] / cnt, acc[4] / cnt, acc[5] / cnt,
                   acc[6] / cnt, acc[7] / cnt,
                   (acc[1] + acc[2] + acc[3] + acc[4] + acc[5] + acc[6] + acc[7]) / cnt, cnt);
  }
  return e;
}

}  // namespace ctri
