// factor.h -- host fp64 pre-factorisation ("the construction of
// L^, D^, U^ and D_i does not require the right-hand-side ... the original
// matrix can be pre-factorized").  Pure host code, no CUDA.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace ctri {

struct Bands {
  double l, d, u;  // A[i,i-1], A[i,i], A[i,i+1]
};

// Outcome of a factorisation step: 0 ok, else a ctri_status value.
struct FactorError {
  int code = 0;
  std::string detail;
};

// Pivot guard: |pivot| < 1e-13 * max|band| trips CTRI_ERR_SINGULAR.
double pivot_threshold(const Bands& b);

// Thomas factors of the acyclic N x N block with constant bands:
//   den[0] = d, den[k] = d - l*cp[k-1], cp[k] = u/den[k].
// Forward:  g_k = (r_k - l g_{k-1}) * inv_den[k];  backward: y_k = g_k - cp[k] y_{k+1}.
struct Thomas {
  std::vector<double> cp, inv_den;
};
bool thomas_factor(int64_t N, const Bands& b, Thomas* out, FactorError* err);
// Solve in place with the factors (host, one column).
void thomas_solve(const Thomas& t, const Bands& b, std::vector<double>& r);

// Partition tables of a block of N interior rows (Eqs. Si, Ri):
//   S = D^{-1}(l e_0), R = D^{-1}(u e_{N-1});
// reduced-row coefficients (Eqs. Li_hat, Di_hat, Ui_hat) for uniform partitions:
//   L^ = -l S[N-1], D^ = d - l R[N-1] - u S[0], U^ = -u R[0].
struct Partition {
  Thomas th;
  std::vector<double> S, R;
  double Lh = 0, Dh = 0, Uh = 0;
};
bool partition_factor(int64_t N, const Bands& b, Partition* out, FactorError* err);

// Rows per slab end where |S[k]| or |R[k]| exceeds 2^-64 (reading R15);
// returns N if the two windows would overlap (then every row is touched).
int64_t backsub_window(const Partition& p);

// PCR reduction coefficients on a P-row tridiagonal system with per-row
// (L, D, U), cyclic (P a power of two, last stage folds the wrapped couplings
// into the diagonal) or acyclic.  alpha/gamma are stage-major [stages][P].
struct PcrTables {
  int P = 0, stages = 0;
  bool cyclic = true;
  std::vector<double> alpha, gamma, inv;
};
bool pcr_factor(int P, bool cyclic, const std::vector<double>& L, const std::vector<double>& D,
                const std::vector<double>& U, double guard, PcrTables* out, FactorError* err);

// Reduced-system schedule executed per batch column by the ranks (one row each):
//   step s, rank i:  v_i <- w * v_i - c[0] * v_{src[0]} - c[1] * v_{src[1]}
// with synchronous semantics (sources read before the step's updates).  Built from PCR steps
// for power-of-two cyclic and all acyclic systems, and from the paper's
// detach / PCR / fold / reattach procedure (worked 11x11 example P:294) for cyclic
// systems of any other dimension.  All coefficients are RHS-independent.
enum StepKind { kStepDetach = 0, kStepPcr = 1, kStepFold = 2, kStepReattach = 3 };
struct SchedEntry {
  double w = 1.0;
  int src[2] = {-1, -1};
  double c[2] = {0.0, 0.0};
};
struct Schedule {
  int P = 0;
  bool cyclic = true;
  std::vector<int> kind;                       // per step
  std::vector<std::vector<SchedEntry>> steps;  // [step][row]
  std::vector<std::vector<int>> detached;      // rows detached at each detach level
  int pcr_stages = 0, detach_stages = 0, detached_rows = 0;
};
bool reduced_schedule(int P, bool cyclic, const std::vector<double>& L, const std::vector<double>& D,
                      const std::vector<double>& U, double guard, Schedule* out, FactorError* err);

// Dense inverse of the P x P reduced matrix A^ (rows L/D/U, cyclic corners; couplings that
// coincide for P <= 2 add up), Gauss-Jordan with partial pivoting, row-major [P][P].  Used by the
// all-gather reduced solve: x~_i = sum_r (A^{-1})_{ir} b^_r.
bool reduced_inverse(int P, bool cyclic, const std::vector<double>& L, const std::vector<double>& D,
                     const std::vector<double>& U, double guard, std::vector<double>* inv,
                     FactorError* err);

// ---- pentadiagonal (r = 2; "for a penta-diagonal system D~_i is 2x2") ----
// Bands (e, l, d, u, f) = (A[i,i-2], A[i,i-1], A[i,i], A[i,i+1], A[i,i+2]).  A partition of n
// rows: rows 0, 1 are the interface x~_i (r = 2 unknowns), rows 2..n-1 the interior (N = n-2).
// Interior block D (acyclic pentadiagonal) = L U without pivoting:
//   lam2[k] = e / mu[k-2],  lam1[k] = (l - lam2[k] nu1[k-2]) / mu[k-1],
//   mu[k] = d - lam1[k] nu1[k-1] - lam2[k] f,  nu1[k] = u - lam1[k] f;
//   forward  z_k = b_k - lam1[k] z_{k-1} - lam2[k] z_{k-2},
//   backward y_k = (z_k - nu1[k] y_{k+1} - f y_{k+2}) / mu[k]          (Eq. yi)
// Couplings (Eqs. Si, Ri with r = 2): S = D^{-1} L, L = [e l; 0 e; 0 ...] (rows 0, 1),
// R = D^{-1} U, U = [... ; f 0; u f] (rows N-2, N-1), stored as columns S0, S1, R0, R1.
// 2x2 reduced blocks (Eqs. Li_hat..Ui_hat), row-major:
//   L^ = -L~ S,  D^ = D~ - L~ R - U~ S,  U^ = -U~ R,  D~ = [d u; l d],
//   L~ = rows (e y[N-2] + l y[N-1], e y[N-1]) of the previous interior, U~ = rows
//   (f y[0], u y[0] + f y[1]) of the own interior.
struct Penta {
  int64_t N = 0;
  std::vector<double> lam1, lam2, nu1, inv_mu;
  std::vector<double> S0, S1, R0, R1;
  double Lh[4] = {0, 0, 0, 0}, Dh[4] = {0, 0, 0, 0}, DhFirst[4] = {0, 0, 0, 0}, Uh[4] = {0, 0, 0, 0};
};
bool penta_factor(int64_t N, const double bd[5], Penta* out, FactorError* err);
// rows per end where some |S| or |R| entry exceeds 2^-64 (reading R15 with r = 2); N if they overlap
int64_t penta_window(const Penta& p);
// dense inverse of the 2P x 2P block-tridiagonal reduced matrix (2x2 blocks; cyclic corners,
// coinciding couplings add up; acyclic: first block row uses DhFirst, no L^ / U^ at the ends)
bool penta_reduced_inverse(int P, bool cyclic, const Penta& pt, double guard, std::vector<double>* inv,
                           FactorError* err);

// Block (2x2) PCR on the pentadiagonal reduced system (P:346 with r = 2): for stage k, s = 2^k,
//   alpha_i = L_i D_{i-s}^{-1},  gamma_i = U_i D_{i+s}^{-1}   (partners i -+ s, mod P if cyclic)
//   b_i <- b_i - alpha_i b_{i-s} - gamma_i b_{i+s}
//   D_i <- D_i - alpha_i U_{i-s} - gamma_i L_{i+s},  L_i <- -alpha_i L_{i-s},  U_i <- -gamma_i U_{i+s}
// Cyclic P = 2^q: after q stages the couplings point back at row i and are folded,
// x~_i = (L_i + D_i + U_i)^{-1} b_i (reading R3 in block form); acyclic: ceil(log2 P) stages,
// x~_i = D_i^{-1} b_i.  Tables are row-major 2x2: alpha / gamma [stage][row][4], fold [row][4].
struct PentaPcr {
  int P = 0, stages = 0;
  bool cyclic = true;
  std::vector<double> alpha, gamma, fold;
};
bool penta_block_pcr(int P, bool cyclic, const Penta& pt, double guard, PentaPcr* out, FactorError* err);
// the same with per-row 2x2 blocks L, D, U ([P][4] row-major each; out-of-range couplings of an
// acyclic system must be zero) -- e.g. the chunk-head systems of the on-chip pentadiagonal
// solve, whose first row may be a decoupled dummy
bool penta_block_pcr_rows(int P, bool cyclic, std::vector<double> L, std::vector<double> D,
                          std::vector<double> U, double guard, PentaPcr* out, FactorError* err);

// The pentadiagonal reduced system as a step schedule with 2x2 blocks (the block form of
// reduced_schedule): every step is  v_i <- W v_i - C0 u_src0 - C1 u_src1  with 2x2 W, C0, C1
// (row-major [4] each; W = I unless stated).  Power-of-two or acyclic P: the block PCR stages
// of penta_block_pcr (a single partner C0 = alpha + gamma when i - s = i + s) and the fold
// W = F_i.  Cyclic P not a power of two: the paper's detach / PCR / fold / reattach (P:271,
// P:294) with 2x2 blocks -- detach: row y <- y - U_y D_z^-1 z, row a <- a - L_a D_z^-1 z;
// reattach: x_z = D_z^-1 (b_z - L_z x_y - U_z x_a).
struct BlockSchedEntry {
  double W[4] = {1.0, 0.0, 0.0, 1.0};
  int src[2] = {-1, -1};
  double C[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
};
struct BlockSchedule {
  int P = 0;
  bool cyclic = true;
  std::vector<int> kind;                            // per step (StepKind)
  std::vector<std::vector<BlockSchedEntry>> steps;  // [step][row]
  int pcr_stages = 0, detach_stages = 0, detached_rows = 0;
};
bool penta_reduced_schedule(int P, bool cyclic, const Penta& pt, double guard, BlockSchedule* out,
                            FactorError* err);

inline bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }
inline int ilog2(int64_t v) {
  int q = 0;
  while ((int64_t(1) << q) < v) ++q;
  return q;
}

}  // namespace ctri
