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

// Gauss-Jordan inverse with partial pivoting of a dense n x n row-major matrix.
static bool dense_inverse(int n, std::vector<double> a, double guard, std::vector<double>* inv,
                          FactorError* err, const char* who) {
  std::vector<double> e((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) e[(size_t)i * n + i] = 1.0;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(a[(size_t)i * n + k]) > std::fabs(a[(size_t)piv * n + k])) piv = i;
    if (!(std::fabs(a[(size_t)piv * n + k]) >= guard))
      return fail(err, kSingular, std::string(who) + ": pivot guard");
    if (piv != k)
      for (int j = 0; j < n; ++j) {
        std::swap(a[(size_t)k * n + j], a[(size_t)piv * n + j]);
        std::swap(e[(size_t)k * n + j], e[(size_t)piv * n + j]);
      }
    const double r = 1.0 / a[(size_t)k * n + k];
    for (int j = 0; j < n; ++j) {
      a[(size_t)k * n + j] *= r;
      e[(size_t)k * n + j] *= r;
    }
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      const double f = a[(size_t)i * n + k];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        a[(size_t)i * n + j] -= f * a[(size_t)k * n + j];
        e[(size_t)i * n + j] -= f * e[(size_t)k * n + j];
      }
    }
  }
  *inv = e;
  return true;
}

bool penta_factor(int64_t N, const double bd[5], Penta* out, FactorError* err) {
  if (N < 4) return fail(err, kInvalid, "penta_factor: interior needs >= 4 rows (n >= 6)");
  const double e = bd[0], l = bd[1], d = bd[2], u = bd[3], f = bd[4];
  double mx = 0;
  for (int k = 0; k < 5; ++k) mx = std::max(mx, std::fabs(bd[k]));
  const double guard = 1e-13 * mx;
  Penta p;
  p.N = N;
  p.lam1.assign(N, 0.0);
  p.lam2.assign(N, 0.0);
  p.nu1.assign(N, 0.0);
  p.inv_mu.assign(N, 0.0);
  std::vector<double> mu(N);
  for (int64_t k = 0; k < N; ++k) {
    const double l2 = k >= 2 ? e / mu[k - 2] : 0.0;
    const double l1 = k >= 1 ? (l - (k >= 2 ? l2 * p.nu1[k - 2] : 0.0)) / mu[k - 1] : 0.0;
    mu[k] = d - (k >= 1 ? l1 * p.nu1[k - 1] : 0.0) - (k >= 2 ? l2 * f : 0.0);
    if (!(std::fabs(mu[k]) >= guard)) return fail(err, kSingular, "penta_factor: pivot guard");
    p.lam1[k] = l1;
    p.lam2[k] = l2;
    p.nu1[k] = u - l1 * f;
    p.inv_mu[k] = 1.0 / mu[k];
  }
  auto solve = [&](std::vector<double> r) {  // D^{-1} r with the factors above
    for (int64_t k = 0; k < N; ++k)
      r[k] -= (k >= 1 ? p.lam1[k] * r[k - 1] : 0.0) + (k >= 2 ? p.lam2[k] * r[k - 2] : 0.0);
    for (int64_t k = N - 1; k >= 0; --k)
      r[k] = (r[k] - (k + 1 < N ? p.nu1[k] * r[k + 1] : 0.0) - (k + 2 < N ? f * r[k + 2] : 0.0)) *
             p.inv_mu[k];
    return r;
  };
  std::vector<double> v(N, 0.0);
  v[0] = e;
  p.S0 = solve(v);  // coefficient of x~_i[0]: interior row 0 (slab row 2) has e
  v.assign(N, 0.0);
  v[0] = l;
  v[1] = e;
  p.S1 = solve(v);  // x~_i[1]: slab rows 2 (l) and 3 (e)
  v.assign(N, 0.0);
  v[N - 2] = f;
  v[N - 1] = u;
  p.R0 = solve(v);  // x~_{i+1}[0]: slab rows n-2 (f) and n-1 (u)
  v.assign(N, 0.0);
  v[N - 1] = f;
  p.R1 = solve(v);  // x~_{i+1}[1]: slab row n-1 (f)
  const std::vector<double>* S[2] = {&p.S0, &p.S1};
  const std::vector<double>* R[2] = {&p.R0, &p.R1};
  for (int c = 0; c < 2; ++c) {
    const std::vector<double>& s = *S[c];
    const std::vector<double>& r = *R[c];
    p.Lh[0 * 2 + c] = -(e * s[N - 2] + l * s[N - 1]);
    p.Lh[1 * 2 + c] = -(e * s[N - 1]);
    const double LR0 = e * r[N - 2] + l * r[N - 1], LR1 = e * r[N - 1];
    const double US0 = f * s[0], US1 = u * s[0] + f * s[1];
    const double Dt0 = c == 0 ? d : u, Dt1 = c == 0 ? l : d;  // D~ = [d u; l d]
    p.Dh[0 * 2 + c] = Dt0 - LR0 - US0;
    p.Dh[1 * 2 + c] = Dt1 - LR1 - US1;
    p.DhFirst[0 * 2 + c] = Dt0 - US0;  // acyclic partition 0: no previous interior
    p.DhFirst[1 * 2 + c] = Dt1 - US1;
    p.Uh[0 * 2 + c] = -(f * r[0]);
    p.Uh[1 * 2 + c] = -(u * r[0] + f * r[1]);
  }
  *out = std::move(p);
  return true;
}

int64_t penta_window(const Penta& p) {
  const double eps = std::ldexp(1.0, -64);
  int64_t lo = 0, hi = 0;  // rows from the start / end with a non-negligible entry
  for (int64_t k = 0; k < p.N; ++k)
    if (std::fabs(p.S0[k]) > eps || std::fabs(p.S1[k]) > eps) lo = k + 1;
  for (int64_t k = 0; k < p.N; ++k)
    if (std::fabs(p.R0[k]) > eps || std::fabs(p.R1[k]) > eps) {
      hi = p.N - k;
      break;
    }
  const int64_t W = std::max(lo <= p.N / 2 ? lo : p.N, hi <= p.N / 2 ? hi : p.N);
  return 2 * W >= p.N ? p.N : W;
}

bool penta_reduced_inverse(int P, bool cyclic, const Penta& pt, double guard, std::vector<double>* inv,
                           FactorError* err) {
  if (P < 1) return fail(err, kInvalid, "penta_reduced_inverse: P < 1");
  const int n = 2 * P;
  std::vector<double> a((size_t)n * n, 0.0);
  auto add = [&](int bi, int bj, const double* blk) {
    for (int r = 0; r < 2; ++r)
      for (int c = 0; c < 2; ++c) a[(size_t)(2 * bi + r) * n + 2 * bj + c] += blk[r * 2 + c];
  };
  for (int i = 0; i < P; ++i) {
    add(i, i, (cyclic || i > 0) ? pt.Dh : pt.DhFirst);
    if (cyclic || i > 0) add(i, (i + P - 1) % P, pt.Lh);
    if (cyclic || i < P - 1) add(i, (i + 1) % P, pt.Uh);
  }
  return dense_inverse(n, a, guard, inv, err, "penta_reduced_inverse");
}

// 2x2 helpers (row-major)
static void mm2(const double* a, const double* b, double* o) {
  const double t0 = a[0] * b[0] + a[1] * b[2], t1 = a[0] * b[1] + a[1] * b[3];
  const double t2 = a[2] * b[0] + a[3] * b[2], t3 = a[2] * b[1] + a[3] * b[3];
  o[0] = t0, o[1] = t1, o[2] = t2, o[3] = t3;
}
static bool inv2(const double* a, double guard, double* o) {
  const double det = a[0] * a[3] - a[1] * a[2];
  const double sc = std::max(std::max(std::fabs(a[0]), std::fabs(a[1])), std::max(std::fabs(a[2]), std::fabs(a[3])));
  if (!(std::fabs(det) >= guard * sc)) return false;
  const double r = 1.0 / det;
  const double t0 = a[3] * r, t1 = -a[1] * r, t2 = -a[2] * r, t3 = a[0] * r;
  o[0] = t0, o[1] = t1, o[2] = t2, o[3] = t3;
  return true;
}

bool penta_block_pcr(int P, bool cyclic, const Penta& pt, double guard, PentaPcr* out, FactorError* err) {
  if (P < 2) return fail(err, kInvalid, "penta_block_pcr: P < 2");
  std::vector<double> L(4 * (size_t)P), D(4 * (size_t)P), U(4 * (size_t)P);
  for (int i = 0; i < P; ++i) {
    const bool lft = cyclic || i > 0, rgt = cyclic || i < P - 1;
    for (int e = 0; e < 4; ++e) {
      L[4 * i + e] = lft ? pt.Lh[e] : 0.0;
      D[4 * i + e] = lft ? pt.Dh[e] : pt.DhFirst[e];
      U[4 * i + e] = rgt ? pt.Uh[e] : 0.0;
    }
  }
  return penta_block_pcr_rows(P, cyclic, L, D, U, guard, out, err);
}

bool penta_block_pcr_rows(int P, bool cyclic, std::vector<double> L, std::vector<double> D,
                          std::vector<double> U, double guard, PentaPcr* out, FactorError* err) {
  if (P < 1) return fail(err, kInvalid, "penta_block_pcr: P < 1");
  if (cyclic && !is_pow2(P)) return fail(err, kUnsupported, "penta_block_pcr: cyclic P must be a power of two");
  PentaPcr t;
  t.P = P;
  t.cyclic = cyclic;
  const int q = ilog2(P);  // cyclic: log2 P; acyclic: ceil(log2 P)
  for (int k = 0; k < q; ++k) {
    const int s = 1 << k;
    std::vector<double> nL(L.size()), nD(D.size()), nU(U.size()), al(4 * (size_t)P, 0.0), ga(4 * (size_t)P, 0.0);
    for (int i = 0; i < P; ++i) {
      int im = i - s, ip = i + s;
      if (cyclic) {
        im = ((im % P) + P) % P;
        ip = ip % P;
      } else {
        if (im < 0) im = -1;
        if (ip >= P) ip = -1;
      }
      double Di[4], a[4] = {0, 0, 0, 0}, g[4] = {0, 0, 0, 0}, tmp[4];
      for (int e = 0; e < 4; ++e) Di[e] = D[4 * i + e];
      double Ln[4] = {0, 0, 0, 0}, Un[4] = {0, 0, 0, 0};
      if (im >= 0) {
        double inv[4];
        if (!inv2(&D[4 * im], guard, inv)) return fail(err, kSingular, "penta_block_pcr: pivot guard");
        mm2(&L[4 * i], inv, a);
        mm2(a, &U[4 * im], tmp);
        for (int e = 0; e < 4; ++e) Di[e] -= tmp[e];
        mm2(a, &L[4 * im], Ln);
        for (int e = 0; e < 4; ++e) Ln[e] = -Ln[e];
      }
      if (ip >= 0) {
        double inv[4];
        if (!inv2(&D[4 * ip], guard, inv)) return fail(err, kSingular, "penta_block_pcr: pivot guard");
        mm2(&U[4 * i], inv, g);
        mm2(g, &L[4 * ip], tmp);
        for (int e = 0; e < 4; ++e) Di[e] -= tmp[e];
        mm2(g, &U[4 * ip], Un);
        for (int e = 0; e < 4; ++e) Un[e] = -Un[e];
      }
      for (int e = 0; e < 4; ++e) {
        nD[4 * i + e] = Di[e];
        nL[4 * i + e] = Ln[e];
        nU[4 * i + e] = Un[e];
        al[4 * i + e] = a[e];
        ga[4 * i + e] = g[e];
      }
    }
    L.swap(nL);
    D.swap(nD);
    U.swap(nU);
    t.alpha.insert(t.alpha.end(), al.begin(), al.end());
    t.gamma.insert(t.gamma.end(), ga.begin(), ga.end());
  }
  t.stages = q;
  t.fold.assign(4 * (size_t)P, 0.0);
  for (int i = 0; i < P; ++i) {
    double m[4];
    for (int e = 0; e < 4; ++e) m[e] = D[4 * i + e] + (cyclic ? L[4 * i + e] + U[4 * i + e] : 0.0);
    if (!inv2(m, guard, &t.fold[4 * (size_t)i])) return fail(err, kSingular, "penta_block_pcr: fold pivot guard");
  }
  *out = std::move(t);
  return true;
}

bool penta_reduced_schedule(int P, bool cyclic, const Penta& pt, double guard, BlockSchedule* out,
                            FactorError* err) {
  *out = BlockSchedule();
  out->P = P;
  out->cyclic = cyclic;
  if (P < 1) return fail(err, kInvalid, "penta_reduced_schedule: P < 1");
  auto sub2 = [](double* a, const double* b) {
    for (int e = 0; e < 4; ++e) a[e] -= b[e];
  };
  auto neg2 = [](double* a) {
    for (int e = 0; e < 4; ++e) a[e] = -a[e];
  };
  if (!cyclic || is_pow2(P)) {  // block PCR stages, then the fold
    if (P == 1) {
      PentaPcr t;
      std::vector<double> L(pt.Lh, pt.Lh + 4), D(cyclic ? pt.Dh : pt.DhFirst, (cyclic ? pt.Dh : pt.DhFirst) + 4),
          U(pt.Uh, pt.Uh + 4);
      if (!cyclic) L.assign(4, 0.0), U.assign(4, 0.0);
      if (!penta_block_pcr_rows(1, cyclic, L, D, U, guard, &t, err)) return false;
      std::vector<BlockSchedEntry> fold(1);
      std::copy(t.fold.begin(), t.fold.begin() + 4, fold[0].W);
      out->kind.push_back(kStepFold);
      out->steps.push_back(fold);
      return true;
    }
    PentaPcr t;
    if (!penta_block_pcr(P, cyclic, pt, guard, &t, err)) return false;
    for (int k = 0; k < t.stages; ++k) {
      const int s = 1 << k;
      std::vector<BlockSchedEntry> st(P);
      for (int i = 0; i < P; ++i) {
        int im = i - s, ip = i + s;
        if (cyclic) {
          im = ((im % P) + P) % P;
          ip = ip % P;
        } else {
          if (im < 0) im = -1;
          if (ip >= P) ip = -1;
        }
        const double* a = &t.alpha[((size_t)k * P + i) * 4];
        const double* g = &t.gamma[((size_t)k * P + i) * 4];
        if (im >= 0 && im == ip) {  // single partner (s = P/2)
          st[i].src[0] = im;
          for (int e = 0; e < 4; ++e) st[i].C[0][e] = a[e] + g[e];
        } else {
          if (im >= 0) { st[i].src[0] = im; std::copy(a, a + 4, st[i].C[0]); }
          if (ip >= 0) { st[i].src[1] = ip; std::copy(g, g + 4, st[i].C[1]); }
        }
      }
      out->kind.push_back(kStepPcr);
      out->steps.push_back(st);
    }
    std::vector<BlockSchedEntry> fold(P);
    for (int i = 0; i < P; ++i) std::copy(&t.fold[4 * (size_t)i], &t.fold[4 * (size_t)i] + 4, fold[i].W);
    out->kind.push_back(kStepFold);
    out->steps.push_back(fold);
    out->pcr_stages = t.stages;
    return true;
  }
  // ---- cyclic, P not a power of two: detach / PCR / fold / reattach with 2x2 blocks ----
  std::vector<double> Lc(4 * (size_t)P), Dc(4 * (size_t)P), Uc(4 * (size_t)P);
  for (int i = 0; i < P; ++i)
    for (int e = 0; e < 4; ++e) {
      Lc[4 * i + e] = pt.Lh[e];
      Dc[4 * i + e] = pt.Dh[e];
      Uc[4 * i + e] = pt.Uh[e];
    }
  std::vector<std::vector<int>> subs(1);
  for (int i = 0; i < P; ++i) subs[0].push_back(i);
  struct Det { int z, y, a; double Lz[4], Dz[4], Uz[4]; };
  std::vector<std::vector<Det>> levels;
  auto inv = [&](const double* m, double* o) -> bool {
    if (!inv2(m, guard, o)) return fail(err, kSingular, "penta_reduced_schedule: pivot guard");
    return true;
  };
  while (subs[0].size() > 1) {
    const int d = (int)subs[0].size();
    if (d % 2) {  // detach the last row of every sub-system
      std::vector<BlockSchedEntry> st(P);
      std::vector<Det> lv;
      for (auto& sub : subs) {
        const int z = sub[d - 1], y = sub[d - 2], a = sub[0];
        double iz[4], cy[4], ca[4], tmp[4];
        if (!inv(&Dc[4 * z], iz)) return false;
        mm2(&Uc[4 * y], iz, cy);  // row y: upper block on z
        mm2(&Lc[4 * a], iz, ca);  // row a: lower block on z (cyclic wrap)
        st[y].src[0] = z;
        std::copy(cy, cy + 4, st[y].C[0]);
        st[a].src[0] = z;
        std::copy(ca, ca + 4, st[a].C[0]);
        Det t;
        t.z = z, t.y = y, t.a = a;
        std::copy(&Lc[4 * z], &Lc[4 * z] + 4, t.Lz);
        std::copy(&Dc[4 * z], &Dc[4 * z] + 4, t.Dz);
        std::copy(&Uc[4 * z], &Uc[4 * z] + 4, t.Uz);
        lv.push_back(t);
        mm2(cy, &Lc[4 * z], tmp);  // y - cy z: z's lower block sits on y, its upper on a
        sub2(&Dc[4 * y], tmp);
        double nUy[4];
        mm2(cy, &Uc[4 * z], nUy);
        neg2(nUy);
        mm2(ca, &Uc[4 * z], tmp);  // a - ca z: z's upper block sits on a, its lower on y
        sub2(&Dc[4 * a], tmp);
        double nLa[4];
        mm2(ca, &Lc[4 * z], nLa);
        neg2(nLa);
        std::copy(nUy, nUy + 4, &Uc[4 * y]);  // y's next row is now a
        std::copy(nLa, nLa + 4, &Lc[4 * a]);  // a's previous row is now y
        sub.pop_back();
      }
      levels.push_back(lv);
      out->kind.push_back(kStepDetach);
      out->steps.push_back(st);
      out->detach_stages++;
      out->detached_rows += (int)lv.size();
      continue;
    }
    // one block PCR step on every (even) sub-system, then split into even / odd positions
    std::vector<BlockSchedEntry> st(P);
    std::vector<double> nL = Lc, nD = Dc, nU = Uc;
    std::vector<std::vector<int>> next;
    for (auto& sub : subs) {
      for (int k = 0; k < d; ++k) {
        const int i = sub[k], pm = sub[(k + d - 1) % d], pn = sub[(k + 1) % d];
        double im[4], in[4], a[4], g[4], tmp[4];
        if (!inv(&Dc[4 * pm], im) || !inv(&Dc[4 * pn], in)) return false;
        mm2(&Lc[4 * i], im, a);
        mm2(&Uc[4 * i], in, g);
        if (pm == pn) {
          st[i].src[0] = pm;
          for (int e = 0; e < 4; ++e) st[i].C[0][e] = a[e] + g[e];
        } else {
          st[i].src[0] = pm;
          std::copy(a, a + 4, st[i].C[0]);
          st[i].src[1] = pn;
          std::copy(g, g + 4, st[i].C[1]);
        }
        mm2(a, &Lc[4 * pm], &nL[4 * i]);
        neg2(&nL[4 * i]);
        mm2(g, &Uc[4 * pn], &nU[4 * i]);
        neg2(&nU[4 * i]);
        std::copy(&Dc[4 * i], &Dc[4 * i] + 4, &nD[4 * i]);
        mm2(a, &Uc[4 * pm], tmp);
        sub2(&nD[4 * i], tmp);
        mm2(g, &Lc[4 * pn], tmp);
        sub2(&nD[4 * i], tmp);
      }
      std::vector<int> ev, od;
      for (int k = 0; k < d; ++k) (k % 2 ? od : ev).push_back(sub[k]);
      next.push_back(ev);
      next.push_back(od);
    }
    Lc.swap(nL);
    Dc.swap(nD);
    Uc.swap(nU);
    subs.swap(next);
    out->kind.push_back(kStepPcr);
    out->steps.push_back(st);
    out->pcr_stages++;
  }
  // fold the wrapped couplings of the 1x1-block sub-systems (reading R3 in block form)
  std::vector<BlockSchedEntry> fold(P);
  for (auto& sub : subs) {
    const int i = sub[0];
    double m[4];
    for (int e = 0; e < 4; ++e) m[e] = Lc[4 * i + e] + Dc[4 * i + e] + Uc[4 * i + e];
    if (!inv(m, fold[i].W)) return false;
  }
  out->kind.push_back(kStepFold);
  out->steps.push_back(fold);
  // reattach the detached rows, last level first
  for (int lvl = (int)levels.size() - 1; lvl >= 0; --lvl) {
    std::vector<BlockSchedEntry> st(P);
    for (const Det& t : levels[lvl]) {
      double iz[4];
      if (!inv(t.Dz, iz)) return false;
      std::copy(iz, iz + 4, st[t.z].W);
      st[t.z].src[0] = t.y;
      mm2(iz, t.Lz, st[t.z].C[0]);
      st[t.z].src[1] = t.a;
      mm2(iz, t.Uz, st[t.z].C[1]);
    }
    out->kind.push_back(kStepReattach);
    out->steps.push_back(st);
  }
  return true;
}

bool reduced_inverse(int P, bool cyclic, const std::vector<double>& L, const std::vector<double>& D,
                     const std::vector<double>& U, double guard, std::vector<double>* inv,
                     FactorError* err) {
  if (P < 1 || (int)L.size() != P || (int)D.size() != P || (int)U.size() != P)
    return fail(err, kInvalid, "reduced_inverse: bad sizes");
  std::vector<double> a((size_t)P * P, 0.0), e((size_t)P * P, 0.0);
  for (int i = 0; i < P; ++i) {
    a[(size_t)i * P + i] += D[i];
    if (cyclic || i > 0) a[(size_t)i * P + (i + P - 1) % P] += L[i];
    if (cyclic || i < P - 1) a[(size_t)i * P + (i + 1) % P] += U[i];
    e[(size_t)i * P + i] = 1.0;
  }
  for (int k = 0; k < P; ++k) {
    int piv = k;
    for (int i = k + 1; i < P; ++i)
      if (std::fabs(a[(size_t)i * P + k]) > std::fabs(a[(size_t)piv * P + k])) piv = i;
    if (!(std::fabs(a[(size_t)piv * P + k]) >= guard)) return fail(err, kSingular, "reduced_inverse: pivot guard");
    if (piv != k)
      for (int j = 0; j < P; ++j) {
        std::swap(a[(size_t)k * P + j], a[(size_t)piv * P + j]);
        std::swap(e[(size_t)k * P + j], e[(size_t)piv * P + j]);
      }
    const double r = 1.0 / a[(size_t)k * P + k];
    for (int j = 0; j < P; ++j) {
      a[(size_t)k * P + j] *= r;
      e[(size_t)k * P + j] *= r;
    }
    for (int i = 0; i < P; ++i) {
      if (i == k) continue;
      const double f = a[(size_t)i * P + k];
      if (f == 0.0) continue;
      for (int j = 0; j < P; ++j) {
        a[(size_t)i * P + j] -= f * a[(size_t)k * P + j];
        e[(size_t)i * P + j] -= f * e[(size_t)k * P + j];
      }
    }
  }
  *inv = e;
  return true;
}

bool reduced_schedule(int P, bool cyclic, const std::vector<double>& L0,
                      const std::vector<double>& D0, const std::vector<double>& U0, double guard,
                      Schedule* out, FactorError* err) {
  *out = Schedule();
  out->P = P;
  out->cyclic = cyclic;
  if (P < 1 || (int)L0.size() != P || (int)D0.size() != P || (int)U0.size() != P)
    return fail(err, kInvalid, "reduced_schedule: bad sizes");
  if (!cyclic || is_pow2(P)) {  // stride PCR (pcr_factor), then the final scaling
    PcrTables t;
    if (!pcr_factor(P, cyclic, L0, D0, U0, guard, &t, err)) return false;
    const int q = t.stages;
    for (int k = 0; k < q; ++k) {
      const int s = 1 << k;
      std::vector<SchedEntry> st(P);
      for (int c = 0; c < P; ++c) {
        int lm = c - s, lp = c + s;
        if (cyclic) {
          lm = ((lm % P) + P) % P;
          lp = lp % P;
        } else {
          if (lm < 0) lm = -1;
          if (lp >= P) lp = -1;
        }
        const double a = t.alpha[(size_t)k * P + c], g = t.gamma[(size_t)k * P + c];
        if (lm >= 0 && lm == lp) {  // single partner (s = P/2)
          st[c].src[0] = lm;
          st[c].c[0] = a + g;
        } else {
          if (lm >= 0) { st[c].src[0] = lm; st[c].c[0] = a; }
          if (lp >= 0) { st[c].src[1] = lp; st[c].c[1] = g; }
        }
      }
      out->kind.push_back(kStepPcr);
      out->steps.push_back(st);
    }
    std::vector<SchedEntry> fold(P);
    for (int c = 0; c < P; ++c) fold[c].w = t.inv[c];
    out->kind.push_back(kStepFold);
    out->steps.push_back(fold);
    out->pcr_stages = q;
    return true;
  }
  // ---- cyclic, P not a power of two: detach / PCR / fold / reattach ----
  // Every row keeps coefficients on its previous (Lc) and next (Uc) row within its current
  // cyclic sub-system; the two may alias (dimension 2).
  std::vector<double> Lc = L0, Dc = D0, Uc = U0;
  std::vector<std::vector<int>> subs(1);
  for (int i = 0; i < P; ++i) subs[0].push_back(i);
  struct Det { int z, y, a; double Lz, Dz, Uz; };
  std::vector<std::vector<Det>> levels;
  auto check = [&](double v) -> bool {
    if (!(std::fabs(v) >= guard)) return fail(err, kSingular, "reduced_schedule: pivot guard");
    return true;
  };
  while (subs[0].size() > 1) {
    const int d = (int)subs[0].size();
    if (d % 2) {  // detach the last row of every sub-system
      std::vector<SchedEntry> st(P);
      std::vector<Det> lv;
      std::vector<int> rows;
      for (auto& sub : subs) {
        const int z = sub[d - 1], y = sub[d - 2], a = sub[0];
        if (!check(Dc[z])) return false;
        const double cy = Uc[y] / Dc[z];  // row y: upper off-diagonal on z
        const double ca = Lc[a] / Dc[z];  // row a: lower off-diagonal on z (cyclic wrap)
        st[y].src[0] = z;
        st[y].c[0] = cy;
        st[a].src[0] = z;
        st[a].c[0] = ca;
        lv.push_back(Det{z, y, a, Lc[z], Dc[z], Uc[z]});
        rows.push_back(z);
        // row y - cy * row z: z's lower entry sits on y, its upper entry on a
        Dc[y] -= cy * Lc[z];
        const double newUy = -cy * Uc[z];
        // row a - ca * row z: z's upper entry sits on a, its lower entry on y
        Dc[a] -= ca * Uc[z];
        const double newLa = -ca * Lc[z];
        Uc[y] = newUy;  // y's next row is now a ("placed in the last column")
        Lc[a] = newLa;  // a's previous row is now y
        sub.pop_back();
      }
      levels.push_back(lv);
      out->detached.push_back(rows);
      out->kind.push_back(kStepDetach);
      out->steps.push_back(st);
      out->detach_stages++;
      out->detached_rows += (int)lv.size();
      continue;
    }
    // one PCR step on every (even) sub-system, then split into even / odd positions
    std::vector<SchedEntry> st(P);
    std::vector<double> nL = Lc, nD = Dc, nU = Uc;
    std::vector<std::vector<int>> next;
    for (auto& sub : subs) {
      for (int k = 0; k < d; ++k) {
        const int i = sub[k], pm = sub[(k + d - 1) % d], pn = sub[(k + 1) % d];
        if (!check(Dc[pm]) || !check(Dc[pn])) return false;
        const double a = Lc[i] / Dc[pm], g = Uc[i] / Dc[pn];
        if (pm == pn) {
          st[i].src[0] = pm;
          st[i].c[0] = a + g;
        } else {
          st[i].src[0] = pm;
          st[i].c[0] = a;
          st[i].src[1] = pn;
          st[i].c[1] = g;
        }
        // row pm: Lc on sub[k-2], Uc on i; row pn: Lc on i, Uc on sub[k+2]
        nL[i] = -a * Lc[pm];
        nU[i] = -g * Uc[pn];
        nD[i] = Dc[i] - a * Uc[pm] - g * Lc[pn];
      }
      std::vector<int> ev, od;
      for (int k = 0; k < d; ++k) (k % 2 ? od : ev).push_back(sub[k]);
      next.push_back(ev);
      next.push_back(od);
    }
    Lc.swap(nL);
    Dc.swap(nD);
    Uc.swap(nU);
    subs.swap(next);
    out->kind.push_back(kStepPcr);
    out->steps.push_back(st);
    out->pcr_stages++;
  }
  // fold the wrapped couplings of the 1x1 sub-systems into the diagonal (R3)
  std::vector<SchedEntry> fold(P);
  for (auto& sub : subs) {
    const int i = sub[0];
    const double dd = Lc[i] + Dc[i] + Uc[i];
    if (!check(dd)) return false;
    fold[i].w = 1.0 / dd;
  }
  out->kind.push_back(kStepFold);
  out->steps.push_back(fold);
  // reattach the detached rows, last level first (rows 9, 10 then row 11)
  for (int lvl = (int)levels.size() - 1; lvl >= 0; --lvl) {
    std::vector<SchedEntry> st(P);
    for (const Det& t : levels[lvl]) {
      st[t.z].w = 1.0 / t.Dz;
      st[t.z].src[0] = t.y;
      st[t.z].c[0] = t.Lz / t.Dz;
      st[t.z].src[1] = t.a;
      st[t.z].c[1] = t.Uz / t.Dz;
    }
    out->kind.push_back(kStepReattach);
    out->steps.push_back(st);
  }
  return true;
}

}  // namespace ctri
