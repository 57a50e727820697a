/*
 * ctri_oracle.c -- CPU ORACLE for the batched cyclic tridiagonal solve.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path (the CUDA library
 * under paper_2101_02286_b200/) links, includes or calls this file.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  It shares no code, tables or constants with
 * the GPU path.
 *
 * What it computes (plain definitions, fp64, plain loops):
 *
 *   oracle_cyclic_solve   x = A^{-1} b for every batch column of a right-layout
 *                         3D grid, A the cyclic tridiagonal matrix with constant
 *                         bands (l, dg, u) = (A[i,i-1], A[i,i], A[i,i+1]),
 *                         corners A[0,N-1] = l, A[N-1,0] = u.
 *                         PAPER.md P:5 ("cyclic tridiagonal system with bands
 *                         B[1/3,1,1/3]", solved 256^2 times in parallel); the
 *                         paper's partition method returns exactly A^{-1} b for
 *                         any partition count (block-LU argument P:254),
 *                         so the oracle is that definition, computed by a
 *                         DIFFERENT textbook direct method: the Thomas algorithm
 *                         with the Sherman-Morrison cyclic correction
 *                         (Numerical Recipes sec. 2.7 "cyclic", gamma = -diag),
 *                         per SURVEY.md sec. 8(c) O-SOLVE.  No partitioning, no PCR.
 *
 *   oracle_acyclic_solve  same, non-periodic A (corners zero): plain Thomas.
 *                         Used for the acyclic variant.
 *
 *   oracle_rhs_stencil    b_j = a (f_{j+1}-f_{j-1})/(2h) + bc (f_{j+2}-f_{j-2})/(4h),
 *                         periodic wrap.  PAPER.md P:65-67 (Lele's collocated
 *                         compact first derivative; a = 14/9, bc = 1/9 are the
 *                         caller's inputs, reading R8).
 *
 *   oracle_rhs_stencil5   b_j = sum_{k=-2..2} c_k f_{(j+k) mod N}: the general
 *                         five-point right-hand side of a compact scheme with
 *                         periodic wrap.  Covers the staggered sixth-order
 *                         derivative and interpolation of PAPER.md P:202-206
 *                         (half-node values g_i = f_{i+1/2} stored at index i)
 *                         as well as the collocated derivative above.
 *
 *   oracle_penta_solve    x = A^{-1} b with A the PENTADIAGONAL matrix of constant
 *                         bands (e, l, d, u, f) = (A[i,i-2], A[i,i-1], A[i,i],
 *                         A[i,i+1], A[i,i+2]), cyclic (wrapped corners) or not.
 *                         PAPER.md P:212 (bandwidth w = 2r+1, r = 2: "penta-diagonal
 *                         system, D~_i is 2x2"), SURVEY 8(f) N3.  Computed by plain
 *                         banded Gaussian elimination without pivoting (the
 *                         matrices are diagonally dominant) and, for the cyclic
 *                         corners, the Sherman-Morrison-Woodbury identity with a
 *                         rank-4 correction (the textbook generalisation of the
 *                         cyclic Thomas algorithm above).  No partitioning, no PCR.
 *
 *   oracle_deriv          stencil followed by the cyclic solve with bands
 *                         (alpha, 1, alpha): the compact first derivative f'.
 *
 * Layout: a global array of dims (d0, d1, d2), right layout (d2 contiguous),
 * PAPER.md P:5 ("right memory layout ... third index maps to contiguous
 * memory").  Solving along dim `sd` means: for each fixed pair of the other
 * two indices, the N = dims[sd] values along sd form one column.
 * Viewed as (outer, N, inner) with strides (N*inner, inner, 1).
 *
 * Pinned by tests/test_oracle_pins.py: dense Gaussian elimination (numpy /
 * LAPACK dgesv) for N <= 64 with non-symmetric bands, the Fourier-eigenvector
 * closed form, the periodic Green's function closed form, the constant RHS,
 * brute force on N = 3, 4, 5, and the modified wavenumber of the sixth-order
 * compact scheme (golden values in tests/golden/).
 *
 * Return codes: 0 ok, 1 invalid argument.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void layout(const int64_t dims[3], int sd, int64_t* outer, int64_t* n,
                   int64_t* inner) {
  *n = dims[sd];
  *outer = 1;
  *inner = 1;
  for (int k = 0; k < sd; ++k) *outer *= dims[k];
  for (int k = sd + 1; k < 3; ++k) *inner *= dims[k];
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thomas algorithm for the ACYCLIC tridiagonal system with sub-diagonal l,
 * diagonal d[i] (row dependent), super-diagonal u, one column of length N
 * with element stride `st`.  rhs and out may alias.  Plain forward
 * elimination then backward substitution (NR sec. 2.4 "tridag"). */
static void thomas_column(int64_t N, double l, const double* d, double u,
                          const double* rhs, double* out, int64_t st,
                          double* cp /* scratch, N */) {
  double den = d[0];
  cp[0] = u / den;
  out[0] = rhs[0] / den;
  for (int64_t i = 1; i < N; ++i) {
    den = d[i] - l * cp[i - 1];
    cp[i] = u / den;
    out[i * st] = (rhs[i * st] - l * out[(i - 1) * st]) / den;
  }
  for (int64_t i = N - 2; i >= 0; --i) out[i * st] -= cp[i] * out[(i + 1) * st];
}

/* O-SOLVE: cyclic tridiagonal solve of every column.
 *   gamma = -dg;  A' = A with d'_0 = dg - gamma, d'_{N-1} = dg - alpha_c*beta/gamma,
 *   corners removed (beta = A[0,N-1] = l, alpha_c = A[N-1,0] = u);
 *   A' y = b;  A' z = v, v = (gamma, 0, ..., 0, alpha_c);
 *   f = (y_0 + beta*y_{N-1}/gamma) / (1 + z_0 + beta*z_{N-1}/gamma);  x = y - f z. */
int oracle_cyclic_solve(const int64_t dims[3], int sd, const double bands[3],
                        const double* b, double* x) {
  if (!dims || !bands || !b || !x || sd < 0 || sd > 2) return 1;
  int64_t outer, N, inner;
  layout(dims, sd, &outer, &N, &inner);
  if (N < 3 || outer < 1 || inner < 1) return 1;
  const double l = bands[0], dg = bands[1], u = bands[2];
  const double beta = l, alpha_c = u, gamma = -dg;
  if (dg == 0.0) return 1;

  double* dmod = (double*)malloc(sizeof(double) * N);
  double* z = (double*)malloc(sizeof(double) * N);
  double* cp = (double*)malloc(sizeof(double) * N);
  if (!dmod || !z || !cp) { free(dmod); free(z); free(cp); return 1; }
  for (int64_t i = 0; i < N; ++i) dmod[i] = dg;
  dmod[0] = dg - gamma;
  dmod[N - 1] = dg - alpha_c * beta / gamma;
  /* z: A' z = v, column independent, computed once. */
  for (int64_t i = 0; i < N; ++i) z[i] = 0.0;
  z[0] = gamma;
  z[N - 1] = alpha_c;
  thomas_column(N, l, dmod, u, z, z, 1, cp);
  const double zden = 1.0 + z[0] + beta * z[N - 1] / gamma;

  /* Thomas factors (column independent). */
  double* den = (double*)malloc(sizeof(double) * N);
  if (!den) { free(dmod); free(z); free(cp); return 1; }
  den[0] = dmod[0];
  cp[0] = u / den[0];
  for (int64_t i = 1; i < N; ++i) {
    den[i] = dmod[i] - l * cp[i - 1];
    cp[i] = u / den[i];
  }

  const int64_t ncols = outer * inner;
  if (inner == 1) {
    /* solve axis contiguous: one column at a time */
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < ncols; ++c) {
      const double* bc = b + c * N;
      double* xc = x + c * N;
      xc[0] = bc[0] / den[0];
      for (int64_t i = 1; i < N; ++i) xc[i] = (bc[i] - l * xc[i - 1]) / den[i];
      for (int64_t i = N - 2; i >= 0; --i) xc[i] -= cp[i] * xc[i + 1];
      const double f = (xc[0] + beta * xc[N - 1] / gamma) / zden;
      for (int64_t i = 0; i < N; ++i) xc[i] -= f * z[i];
    }
  } else {
    /* strided solve axis: batch-inner loops over blocks of columns */
    const int64_t BLK = 256;
    const int64_t nblk = (inner + BLK - 1) / BLK;
#pragma omp parallel for schedule(static) collapse(2)
    for (int64_t o = 0; o < outer; ++o) {
      for (int64_t kb = 0; kb < nblk; ++kb) {
        const int64_t c0 = kb * BLK;
        const int64_t c1 = (c0 + BLK < inner) ? c0 + BLK : inner;
        const double* bo = b + o * N * inner;
        double* xo = x + o * N * inner;
        for (int64_t c = c0; c < c1; ++c) xo[c] = bo[c] / den[0];
        for (int64_t i = 1; i < N; ++i) {
          const double rden = den[i];
          for (int64_t c = c0; c < c1; ++c)
            xo[i * inner + c] = (bo[i * inner + c] - l * xo[(i - 1) * inner + c]) / rden;
        }
        for (int64_t i = N - 2; i >= 0; --i) {
          const double cpi = cp[i];
          for (int64_t c = c0; c < c1; ++c) xo[i * inner + c] -= cpi * xo[(i + 1) * inner + c];
        }
        double f[256];
        for (int64_t c = c0; c < c1; ++c)
          f[c - c0] = (xo[c] + beta * xo[(N - 1) * inner + c] / gamma) / zden;
        for (int64_t i = 0; i < N; ++i) {
          const double zi = z[i];
          for (int64_t c = c0; c < c1; ++c) xo[i * inner + c] -= f[c - c0] * zi;
        }
      }
    }
  }
  free(den);
  free(dmod);
  free(z);
  free(cp);
  return 0;
}

/* Acyclic variant: corners zero, plain Thomas on every column (N >= 1). */
int oracle_acyclic_solve(const int64_t dims[3], int sd, const double bands[3],
                         const double* b, double* x) {
  if (!dims || !bands || !b || !x || sd < 0 || sd > 2) return 1;
  int64_t outer, N, inner;
  layout(dims, sd, &outer, &N, &inner);
  if (N < 1 || outer < 1 || inner < 1) return 1;
  const double l = bands[0], dg = bands[1], u = bands[2];
  double* d = (double*)malloc(sizeof(double) * N);
  if (!d) return 1;
  for (int64_t i = 0; i < N; ++i) d[i] = dg;
  const int64_t ncols = outer * inner;
#pragma omp parallel
  {
    double* cp = (double*)malloc(sizeof(double) * N);
#pragma omp for schedule(static)
    for (int64_t c = 0; c < ncols; ++c) {
      const int64_t o = c / inner, k = c % inner;
      thomas_column(N, l, d, u, b + o * N * inner + k, x + o * N * inner + k, inner, cp);
    }
    free(cp);
  }
  free(d);
  return 0;
}

/* Collocated compact-derivative RHS stencil, periodic. */
int oracle_rhs_stencil(const int64_t dims[3], int sd, double a, double bc,
                       double h, const double* f, double* rhs) {
  if (!dims || !f || !rhs || sd < 0 || sd > 2 || h == 0.0 || f == rhs) return 1;
  int64_t outer, N, inner;
  layout(dims, sd, &outer, &N, &inner);
  if (N < 5) return 1;
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t o = 0; o < outer; ++o) {
    for (int64_t j = 0; j < N; ++j) {
      const int64_t jp1 = (j + 1) % N, jm1 = (j - 1 + N) % N;
      const int64_t jp2 = (j + 2) % N, jm2 = (j - 2 + N) % N;
      const double* fo = f + o * N * inner;
      double* ro = rhs + o * N * inner + j * inner;
      for (int64_t c = 0; c < inner; ++c) {
        ro[c] = a * (fo[jp1 * inner + c] - fo[jm1 * inner + c]) / (2.0 * h) +
                bc * (fo[jp2 * inner + c] - fo[jm2 * inner + c]) / (4.0 * h);
      }
    }
  }
  return 0;
}

/* Banded Gaussian elimination without pivoting, one column of length N >= 1 (element
 * stride st): rows i hold A[i,i-2..i+2] = (e, l, d, u, f) truncated at the ends.  The
 * work arrays hold the current band entries of every row while columns are eliminated. */
static void penta_column(int64_t N, const double bd[5], const double* rhs, double* out,
                         int64_t st, double* w /* scratch: 6N */) {
  double *s2 = w, *s1 = w + N, *dg = w + 2 * N, *p1 = w + 3 * N, *p2 = w + 4 * N, *r = w + 5 * N;
  for (int64_t i = 0; i < N; ++i) {
    s2[i] = bd[0];
    s1[i] = bd[1];
    dg[i] = bd[2];
    p1[i] = bd[3];
    p2[i] = bd[4];
    r[i] = rhs[i * st];
  }
  for (int64_t k = 0; k + 1 < N; ++k) {  /* eliminate column k from rows k+1, k+2 */
    const double m1 = s1[k + 1] / dg[k];
    dg[k + 1] -= m1 * p1[k];
    if (k + 2 < N) p1[k + 1] -= m1 * p2[k];
    r[k + 1] -= m1 * r[k];
    if (k + 2 < N) {
      const double m2 = s2[k + 2] / dg[k];
      s1[k + 2] -= m2 * p1[k];
      dg[k + 2] -= m2 * p2[k];
      r[k + 2] -= m2 * r[k];
    }
  }
  for (int64_t i = N - 1; i >= 0; --i) {
    double v = r[i];
    if (i + 1 < N) v -= p1[i] * out[(i + 1) * st];
    if (i + 2 < N) v -= p2[i] * out[(i + 2) * st];
    out[i * st] = v / dg[i];
  }
}

/* Gauss-Jordan inverse of a 4x4 matrix with partial pivoting (in place). */
static int inverse4(double a[16]) {
  double e[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
  for (int k = 0; k < 4; ++k) {
    int pv = k;
    for (int i = k + 1; i < 4; ++i)
      if (fabs(a[i * 4 + k]) > fabs(a[pv * 4 + k])) pv = i;
    if (a[pv * 4 + k] == 0.0) return 1;
    for (int j = 0; j < 4; ++j) {
      double t = a[k * 4 + j]; a[k * 4 + j] = a[pv * 4 + j]; a[pv * 4 + j] = t;
      t = e[k * 4 + j]; e[k * 4 + j] = e[pv * 4 + j]; e[pv * 4 + j] = t;
    }
    const double rp = 1.0 / a[k * 4 + k];
    for (int j = 0; j < 4; ++j) { a[k * 4 + j] *= rp; e[k * 4 + j] *= rp; }
    for (int i = 0; i < 4; ++i) {
      if (i == k) continue;
      const double m = a[i * 4 + k];
      for (int j = 0; j < 4; ++j) { a[i * 4 + j] -= m * a[k * 4 + j]; e[i * 4 + j] -= m * e[k * 4 + j]; }
    }
  }
  memcpy(a, e, sizeof(e));
  return 0;
}

/* Pentadiagonal solve of every column.  Acyclic: penta_column.  Cyclic (N >= 5): the six
 * corner entries A[0,N-2] = e, A[0,N-1] = l, A[1,N-1] = e, A[N-2,0] = f, A[N-1,0] = u,
 * A[N-1,1] = f live in rows J = {0, 1, N-2, N-1}, so A = B + E_J V^T with B the banded
 * part, E_J the columns e_j (j in J) and V^T the corner rows.  Woodbury:
 *   y = B^{-1} b,  Z = B^{-1} E_J (once),  M = I + V^T Z (4x4, once),
 *   x = y - Z M^{-1} V^T y. */
int oracle_penta_solve(const int64_t dims[3], int sd, const double bands[5], int cyclic,
                       const double* b, double* x) {
  if (!dims || !bands || !b || !x || sd < 0 || sd > 2) return 1;
  int64_t outer, N, inner;
  layout(dims, sd, &outer, &N, &inner);
  if (N < (cyclic ? 5 : 1) || outer < 1 || inner < 1) return 1;
  const double e = bands[0], l = bands[1], u = bands[3], f = bands[4];
  double* Z = NULL;
  double M[16];
  if (cyclic) {
    Z = (double*)malloc(sizeof(double) * 4 * N);
    double* w = (double*)malloc(sizeof(double) * 7 * N);
    if (!Z || !w) { free(Z); free(w); return 1; }
    const int64_t J[4] = {0, 1, N - 2, N - 1};
    for (int c = 0; c < 4; ++c) {
      double* unit = w + 6 * N;
      for (int64_t i = 0; i < N; ++i) unit[i] = 0.0;
      unit[J[c]] = 1.0;
      penta_column(N, bands, unit, Z + c * N, 1, w);
    }
    free(w);
    /* V^T z for a column z: the corner rows applied to z */
    for (int c = 0; c < 4; ++c) {
      const double* z = Z + c * N;
      const double vz[4] = {e * z[N - 2] + l * z[N - 1], e * z[N - 1], f * z[0], u * z[0] + f * z[1]};
      for (int rr = 0; rr < 4; ++rr) M[rr * 4 + c] = (rr == c ? 1.0 : 0.0) + vz[rr];
    }
    if (inverse4(M)) { free(Z); return 1; }
  }
  const int64_t ncols = outer * inner;
  int bad = 0;
#pragma omp parallel
  {
    double* w = (double*)malloc(sizeof(double) * 6 * N);
    if (!w) {
#pragma omp atomic write
      bad = 1;
    } else {
#pragma omp for schedule(static)
      for (int64_t t = 0; t < ncols; ++t) {
        const int64_t o = t / inner, c = t % inner;
        const double* bc = b + o * N * inner + c;
        double* xc = x + o * N * inner + c;
        penta_column(N, bands, bc, xc, inner, w);
        if (cyclic) {
          const double vy[4] = {e * xc[(N - 2) * inner] + l * xc[(N - 1) * inner],
                                e * xc[(N - 1) * inner], f * xc[0], u * xc[0] + f * xc[inner]};
          double g[4];
          for (int rr = 0; rr < 4; ++rr)
            g[rr] = M[rr * 4 + 0] * vy[0] + M[rr * 4 + 1] * vy[1] + M[rr * 4 + 2] * vy[2] +
                    M[rr * 4 + 3] * vy[3];
          for (int64_t i = 0; i < N; ++i)
            xc[i * inner] -= Z[i] * g[0] + Z[N + i] * g[1] + Z[2 * N + i] * g[2] + Z[3 * N + i] * g[3];
        }
      }
      free(w);
    }
  }
  free(Z);
  return bad;
}

/* General five-point periodic stencil (PAPER.md P:202-206 schemes): plain definition. */
int oracle_rhs_stencil5(const int64_t dims[3], int sd, const double coef[5], const double* f,
                        double* rhs) {
  if (!dims || !coef || !f || !rhs || sd < 0 || sd > 2 || f == rhs) return 1;
  int64_t outer, N, inner;
  layout(dims, sd, &outer, &N, &inner);
  if (N < 5) return 1;
#pragma omp parallel for schedule(static) collapse(2)
  for (int64_t o = 0; o < outer; ++o) {
    for (int64_t j = 0; j < N; ++j) {
      const double* fo = f + o * N * inner;
      double* ro = rhs + o * N * inner + j * inner;
      for (int64_t c = 0; c < inner; ++c) {
        double acc = 0.0;
        for (int k = -2; k <= 2; ++k) acc += coef[k + 2] * fo[((j + k + N) % N) * inner + c];
        ro[c] = acc;
      }
    }
  }
  return 0;
}

/* Compact first derivative: stencil, then cyclic solve with (alpha, 1, alpha). */
int oracle_deriv(const int64_t dims[3], int sd, double alpha, double a, double bc,
                 double h, const double* f, double* df) {
  if (!dims || !f || !df || f == df) return 1;
  int rc = oracle_rhs_stencil(dims, sd, a, bc, h, f, df);
  if (rc) return rc;
  const double bands[3] = {alpha, 1.0, alpha};
  return oracle_cyclic_solve(dims, sd, bands, df, df);
}
