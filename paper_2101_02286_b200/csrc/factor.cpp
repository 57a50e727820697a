// factor.cpp -- host fp64 pre-factorisation tables.
#include "factor.h"

#include <algorithm>
#include <cmath>
#include <cstdio>

namespace ctri {

static constexpr int kOk = 0, kInvalid = 1, kUnsupported = 2, kSingular = 3;

double pivot_threshold(const Bands& b) {
  double m = std::max(std::fabs(b.l), std::max(std::fabs(b.d), std::fabs(b.u)));
  return 1e-13 * m;
}

static bool fail(FactorError* err, int code, const std::string& msg) {
  if (err) {
    err->code = code;
    err->detail = msg;
  }
  return false;
}

bool thomas_factor(int64_t N, const Bands& b, Thomas* out, FactorError* err) {
  if (N < 1) return fail(err, kInvalid, "thomas_factor: N < 1");
  const double guard = pivot_threshold(b);
  out->cp.assign(N, 0.0);
  out->inv_den.assign(N, 0.0);
  double den = b.d;
  for (int64_t k = 0; k < N; ++k) {
    if (k > 0) den = b.d - b.l * out->cp[k - 1];
    if (!(std::fabs(den) >= guard)) {
      char buf[160];
      std::snprintf(buf, sizeof buf, "pivot guard: |den[%lld]| = %.3e < %.3e", (long long)k,
                    std::fabs(den), guard);
      return fail(err, kSingular, buf);
    }
    out->cp[k] = b.u / den;
    out->inv_den[k] = 1.0 / den;
  }
  return true;
}

void thomas_solve(const Thomas& t, const Bands& b, std::vector<double>& r) {
  const int64_t N = (int64_t)t.cp.size();
  double g = 0.0;
  for (int64_t k = 0; k < N; ++k) {
    g = (r[k] - (k ? b.l * g : 0.0)) * t.inv_den[k];
    r[k] = g;
  }
  for (int64_t k = N - 2; k >= 0; --k) r[k] -= t.cp[k] * r[k + 1];
}

bool partition_factor(int64_t N, const Bands& b, Partition* out, FactorError* err) {
  if (!thomas_factor(N, b, &out->th, err)) return false;
  out->S.assign(N, 0.0);
  out->R.assign(N, 0.0);
  out->S[0] = b.l;      // L_i = l e_0  (first interior row couples to x~_i)
  out->R[N - 1] = b.u;  // U_i = u e_{N-1} (last interior row couples to x~_{i+1})
  thomas_solve(out->th, b, out->S);
  thomas_solve(out->th, b, out->R);
  out->Lh = -b.l * out->S[N - 1];
  out->Dh = b.d - b.l * out->R[N - 1] - b.u * out->S[0];
  out->Uh = -b.u * out->R[0];
  return true;
}

int64_t backsub_window(const Partition& p) {
  const int64_t N = (int64_t)p.S.size();
  const double tau = std::ldexp(1.0, -64);
  int64_t top = 0, bot = 0;
  for (int64_t k = 0; k < N; ++k)
    if (std::fabs(p.S[k]) > tau || std::fabs(p.R[k]) > tau) {
      if (k < N / 2) top = std::max(top, k + 1);
      else bot = std::max(bot, N - k);
    }
  int64_t w = std::max(top, bot);
  if (2 * w >= N) return N;
  return w;
}

bool pcr_factor(int P, bool cyclic, const std::vector<double>& L0, const std::vector<double>& D0,
                const std::vector<double>& U0, double guard, PcrTables* out, FactorError* err) {
  if (P < 1 || (int)L0.size() != P || (int)D0.size() != P || (int)U0.size() != P)
    return fail(err, kInvalid, "pcr_factor: bad sizes");
  if (cyclic && !is_pow2(P))
    return fail(err, kUnsupported,
                "cyclic PCR needs a power-of-two row count (detach/reattach, P:271, not built)");
  std::vector<double> L = L0, D = D0, U = U0;
  if (!cyclic) {
    L[0] = 0.0;
    U[P - 1] = 0.0;
  }
  const int q = ilog2(P);
  out->P = P;
  out->stages = q;
  out->cyclic = cyclic;
  out->alpha.assign((size_t)q * P, 0.0);
  out->gamma.assign((size_t)q * P, 0.0);
  out->inv.assign(P, 0.0);
  auto idx = [&](int c) -> int {  // wrapped or -1 if out of range
    if (cyclic) return ((c % P) + P) % P;
    return (c >= 0 && c < P) ? c : -1;
  };
  std::vector<double> nL(P), nD(P), nU(P);
  for (int k = 0; k < q; ++k) {
    const int s = 1 << k;
    for (int c = 0; c < P; ++c) {
      const int lm = idx(c - s), lp = idx(c + s);
      double a = 0.0, g = 0.0;
      if (lm >= 0 && L[c] != 0.0) {
        if (!(std::fabs(D[lm]) >= guard)) return fail(err, kSingular, "pcr_factor: pivot guard");
        a = L[c] / D[lm];
      }
      if (lp >= 0 && U[c] != 0.0) {
        if (!(std::fabs(D[lp]) >= guard)) return fail(err, kSingular, "pcr_factor: pivot guard");
        g = U[c] / D[lp];
      }
      out->alpha[(size_t)k * P + c] = a;
      out->gamma[(size_t)k * P + c] = g;
      // Row c - a*row(lm) - g*row(lp).  row(lm) = L[lm] on lm-s, D[lm] on lm, U[lm] on lm+s = c;
      // row(lp) = L[lp] on lp-s = c, D[lp] on lp, U[lp] on lp+s.  The new row couples to c-2s
      // and c+2s; in the cyclic case those may alias c itself (folded after the last stage).
      nL[c] = (lm >= 0) ? -a * L[lm] : 0.0;
      nU[c] = (lp >= 0) ? -g * U[lp] : 0.0;
      nD[c] = D[c] - (lm >= 0 ? a * U[lm] : 0.0) - (lp >= 0 ? g * L[lp] : 0.0);
      if (!cyclic) {
        if (c - 2 * s < 0) nL[c] = 0.0;
        if (c + 2 * s >= P) nU[c] = 0.0;
      }
    }
    L.swap(nL);
    D.swap(nD);
    U.swap(nU);
  }
  for (int c = 0; c < P; ++c) {
    // Cyclic: after log2 P stages the couplings point at c +- P == c (fold, R3);
    // P = 1 is the 1x1 closure (L^ + D^ + U^) x~ = b^.
    const double diag = cyclic ? (L[c] + D[c] + U[c]) : D[c];
    if (!(std::fabs(diag) >= guard)) return fail(err, kSingular, "pcr_factor: final pivot guard");
    out->inv[c] = 1.0 / diag;
  }
  return true;
}

}  // namespace ctri
