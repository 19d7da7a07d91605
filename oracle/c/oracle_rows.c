/* ORACLE (test infrastructure only) — plain C row evaluator of the dense
 * Burton-Miller collocation operators, fp64.  Same definition as
 * oracle/dense.py (Eq. (5); collocation at centroids,
 * P:896-906; tier rule = SURVEY §8(c) reading C6), written as plain loops so
 * that the sampled-row oracle of configs 2-5 and the CPU baseline finish in
 * seconds.  Off-diagonal entries only: the self entry (tier T0, closed form,
 * reading C5) is added by oracle/selfterms.py on the Python side.
 * Rows are independent; OpenMP parallelises over rows.  Pinned by agreement
 * with oracle/dense.py (tests/test_oracle_dense.py).  Shares nothing with the
 * CUDA path.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

static const double PI = 3.14159265358979323846;

/* Q3: Strang-Fix 3-point (2/3,1/6,1/6), degree 2 */
static const double Q3_P[3][3] = {{2.0/3, 1.0/6, 1.0/6}, {1.0/6, 2.0/3, 1.0/6}, {1.0/6, 1.0/6, 2.0/3}};
static const double Q3_W[3] = {1.0/3, 1.0/3, 1.0/3};

/* Q6: Dunavant 6-point, degree 4 */
static double Q6_P[6][3];
static double Q6_W[6];
/* Q7: Radon 7-point, degree 5 */
static double Q7_P[7][3];
static double Q7_W[7];
/* T1: Q7 on the depth-3 uniform 1:4 subdivision (448 points) */
static double T1_P[448][3];
static double T1_W[448];
static int rules_ready = 0;

static void sym3(double P[][3], double *W, int at, double a, double w) {
  double b = 1.0 - 2.0 * a;
  double pts[3][3] = {{b, a, a}, {a, b, a}, {a, a, b}};
  for (int q = 0; q < 3; ++q) {
    for (int c = 0; c < 3; ++c) P[at + q][c] = pts[q][c];
    W[at + q] = w;
  }
}

static void subdivide(double tri[3][3], int depth, int *count) {
  if (depth == 0) {
    for (int q = 0; q < 7; ++q) {
      for (int c = 0; c < 3; ++c) {
        double v = 0.0;
        for (int m = 0; m < 3; ++m) v += Q7_P[q][m] * tri[m][c];
        T1_P[*count][c] = v;
      }
      T1_W[*count] = Q7_W[q] / 64.0;
      (*count)++;
    }
    return;
  }
  double ab[3], bc[3], ca[3];
  for (int c = 0; c < 3; ++c) {
    ab[c] = 0.5 * (tri[0][c] + tri[1][c]);
    bc[c] = 0.5 * (tri[1][c] + tri[2][c]);
    ca[c] = 0.5 * (tri[2][c] + tri[0][c]);
  }
  double s[4][3][3];
  for (int c = 0; c < 3; ++c) {
    s[0][0][c] = tri[0][c]; s[0][1][c] = ab[c]; s[0][2][c] = ca[c];
    s[1][0][c] = ab[c]; s[1][1][c] = tri[1][c]; s[1][2][c] = bc[c];
    s[2][0][c] = ca[c]; s[2][1][c] = bc[c]; s[2][2][c] = tri[2][c];
    s[3][0][c] = ab[c]; s[3][1][c] = bc[c]; s[3][2][c] = ca[c];
  }
  for (int t = 0; t < 4; ++t) subdivide(s[t], depth - 1, count);
}

static void init_rules(void) {
  if (rules_ready) return;
  sym3(Q6_P, Q6_W, 0, 0.445948490915965, 0.223381589678011);
  sym3(Q6_P, Q6_W, 3, 0.091576213509771, 0.109951743655322);
  double s15 = sqrt(15.0);
  Q7_P[0][0] = Q7_P[0][1] = Q7_P[0][2] = 1.0 / 3.0;
  Q7_W[0] = 9.0 / 40.0;
  sym3(Q7_P, Q7_W, 1, (6.0 - s15) / 21.0, (155.0 - s15) / 1200.0);
  sym3(Q7_P, Q7_W, 4, (6.0 + s15) / 21.0, (155.0 + s15) / 1200.0);
  double ref[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  int count = 0;
  subdivide(ref, 3, &count);
  rules_ready = 1;
}

/* kind 0: LHS  dG/dn_y + alpha d2G/dn_x dn_y ; kind 1: RHS  G + alpha dG/dn_x
 * (SURVEY App. B formulas). */
static double complex kernel(int kind, const double *x, const double *nx, const double *y,
                             const double *ny, double k, double complex alpha) {
  double d[3] = {x[0] - y[0], x[1] - y[1], x[2] - y[2]};
  double r = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  double complex e = cexp(I * k * r);
  double complex g = e / (4.0 * PI * r);
  double complex gp = e * (I * k * r - 1.0) / (4.0 * PI * r * r);
  double drdnx = (d[0] * nx[0] + d[1] * nx[1] + d[2] * nx[2]) / r;
  if (kind == 1) return g + alpha * gp * drdnx;
  double drdny = -(d[0] * ny[0] + d[1] * ny[1] + d[2] * ny[2]) / r;
  double nxny = nx[0] * ny[0] + nx[1] * ny[1] + nx[2] * ny[2];
  double complex gpp = e * (2.0 - 2.0 * I * k * r - k * k * r * r) / (4.0 * PI * r * r * r);
  double complex hyp = (gpp - gp / r) * drdnx * drdny - gp * nxny / r;
  return gp * drdny + alpha * hyp;
}

static double complex entry(int kind, int64_t i, int64_t j, const double *verts, const double *cen,
                            const double *nrm, const double *area, const double *hmax, double k,
                            double complex alpha) {
  const double *x = cen + 3 * i;
  double dx = x[0] - cen[3 * j], dy = x[1] - cen[3 * j + 1], dz = x[2] - cen[3 * j + 2];
  double rho = sqrt(dx * dx + dy * dy + dz * dz) / hmax[j];
  const double(*P)[3];
  const double *W;
  int nq;
  if (rho >= 3.0) { P = Q3_P; W = Q3_W; nq = 3; }
  else if (rho >= 1.5) { P = (const double(*)[3])Q6_P; W = Q6_W; nq = 6; }
  else { P = (const double(*)[3])T1_P; W = T1_W; nq = 448; }
  const double *v = verts + 9 * j;
  double complex s = 0.0;
  for (int q = 0; q < nq; ++q) {
    double y[3];
    for (int c = 0; c < 3; ++c) y[c] = P[q][0] * v[c] + P[q][1] * v[3 + c] + P[q][2] * v[6 + c];
    s += W[q] * kernel(kind, x, nrm + 3 * i, y, nrm + 3 * j, k, alpha);
  }
  return area[j] * s;
}

/* y[r] = sum_{j != rows[r]} A_{rows[r], j} x_j  (complex interleaved). */
void oracle_matvec_rows(int kind, int64_t n, const double *verts, const double *cen,
                        const double *nrm, const double *area, const double *hmax, double k,
                        double alpha_re, double alpha_im, const double *x, const int64_t *rows,
                        int64_t nrows, double *y) {
  init_rules();
  double complex alpha = alpha_re + I * alpha_im;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t i = rows[r];
    double complex acc = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      double complex xj = x[2 * j] + I * x[2 * j + 1];
      acc += entry(kind, i, j, verts, cen, nrm, area, hmax, k, alpha) * xj;
    }
    y[2 * r] = creal(acc);
    y[2 * r + 1] = cimag(acc);
  }
}

/* out[r*n + j] = A_{rows[r], j} for j != rows[r], 0 on the diagonal. */
void oracle_rows(int kind, int64_t n, const double *verts, const double *cen, const double *nrm,
                 const double *area, const double *hmax, double k, double alpha_re,
                 double alpha_im, const int64_t *rows, int64_t nrows, double *out) {
  init_rules();
  double complex alpha = alpha_re + I * alpha_im;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t i = rows[r];
    for (int64_t j = 0; j < n; ++j) {
      double complex a = 0.0;
      if (j != i) a = entry(kind, i, j, verts, cen, nrm, area, hmax, k, alpha);
      out[2 * (r * n + j)] = creal(a);
      out[2 * (r * n + j) + 1] = cimag(a);
    }
  }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
