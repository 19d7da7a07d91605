// Dense complex fp64 linear algebra for the build (host): one-sided Jacobi
// SVD (for the truncated pseudo-inverses of PAPER.md Eq. (eq_svdg)-(eq_invg),
// P:679-705) and a plain column-major complex GEMM.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "fda_internal.h"

namespace fda {

// C (m×n) = op(A) · B ; op(A) = A (m×kk, lda) or A^H (A stored kk×m, lda).
// C is overwritten.  Serial: callers parallelise over independent products.
void zgemm_cm(int m, int n, int kk, const cd* A, int lda, const cd* B, int ldb, cd* C, int ldc,
              bool conjA_T) {
  if (!conjA_T) {
    for (int j = 0; j < n; ++j) {
      cd* c = C + (size_t)j * ldc;
      for (int i = 0; i < m; ++i) c[i] = 0.0;
      for (int p = 0; p < kk; ++p) {
        const cd b = B[p + (size_t)j * ldb];
        const cd* a = A + (size_t)p * lda;
        for (int i = 0; i < m; ++i) c[i] += a[i] * b;
      }
    }
  } else {
    for (int j = 0; j < n; ++j) {
      const cd* b = B + (size_t)j * ldb;
      for (int i = 0; i < m; ++i) {
        const cd* a = A + (size_t)i * lda;
        cd s = 0.0;
        for (int p = 0; p < kk; ++p) s += std::conj(a[p]) * b[p];
        C[i + (size_t)j * ldc] = s;
      }
    }
  }
}

// One-sided (Hestenes) Jacobi SVD of a column-major m×n complex matrix,
// m >= n.  On exit A holds U (m×n, orthonormal columns for σ > 0), S the
// singular values in descending order and V the n×n unitary factor, so that
// A_in = U diag(S) V^H.  Column pairs are processed in round-robin order so
// that the n/2 rotations of a round are independent (OpenMP).
void svd_jacobi(int m, int n, std::vector<cd>& A, std::vector<double>& S, std::vector<cd>& V) {
  V.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
  const int np = n + (n & 1);
  std::vector<int> idx(np);
  std::iota(idx.begin(), idx.end(), 0);
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 40; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < np - 1; ++round) {
#pragma omp parallel for schedule(static) reduction(+ : rotated)
      for (int kp = 0; kp < np / 2; ++kp) {
        int p = idx[kp], q = idx[np - 1 - kp];
        if (p >= n || q >= n) continue;
        if (p > q) std::swap(p, q);
        cd* ap = A.data() + (size_t)p * m;
        cd* aq = A.data() + (size_t)q * m;
        double alpha = 0, beta = 0;
        cd gamma = 0;
        for (int i = 0; i < m; ++i) {
          alpha += std::norm(ap[i]);
          beta += std::norm(aq[i]);
          gamma += std::conj(ap[i]) * aq[i];
        }
        double ag = std::abs(gamma);
        if (ag <= tol * std::sqrt(alpha * beta) || ag == 0.0) continue;
        ++rotated;
        double zeta = (beta - alpha) / (2.0 * ag);
        double tt = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        double c = 1.0 / std::sqrt(1.0 + tt * tt), s = c * tt;
        cd ph = gamma / ag;  // e^{iφ}
        // [a_p a_q] ← [a_p a_q] [[c, s e^{iφ}], [-s e^{-iφ}, c]]
        for (int i = 0; i < m; ++i) {
          cd x = ap[i], y = aq[i];
          ap[i] = c * x - s * std::conj(ph) * y;
          aq[i] = s * ph * x + c * y;
        }
        cd* vp = V.data() + (size_t)p * n;
        cd* vq = V.data() + (size_t)q * n;
        for (int i = 0; i < n; ++i) {
          cd x = vp[i], y = vq[i];
          vp[i] = c * x - s * std::conj(ph) * y;
          vq[i] = s * ph * x + c * y;
        }
      }
      // rotate idx[1..np-1]
      int last = idx[np - 1];
      for (int k = np - 1; k > 1; --k) idx[k] = idx[k - 1];
      idx[1] = last;
    }
    if (rotated == 0) break;
  }
  std::vector<double> sv(n);
  for (int j = 0; j < n; ++j) {
    double s = 0;
    for (int i = 0; i < m; ++i) s += std::norm(A[(size_t)j * m + i]);
    sv[j] = std::sqrt(s);
  }
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return sv[a] > sv[b]; });
  std::vector<cd> U2((size_t)m * n), V2((size_t)n * n);
  S.resize(n);
  for (int j = 0; j < n; ++j) {
    int o = ord[j];
    S[j] = sv[o];
    double inv = sv[o] > 0 ? 1.0 / sv[o] : 0.0;
    for (int i = 0; i < m; ++i) U2[(size_t)j * m + i] = A[(size_t)o * m + i] * inv;
    for (int i = 0; i < n; ++i) V2[(size_t)j * n + i] = V[(size_t)o * n + i];
  }
  A.swap(U2);
  V.swap(V2);
}

}  // namespace fda

namespace fda {

// Second-stage low-rank factorisation of a reduced M2L matrix (§4.2,
// Eq. (eq_epsk)): K̃ (m×n, column-major) ≈ Û V̂ with Û = U_r S_r
// (m×r) and V̂ = Q_r^H (r×n), truncating σ_i < ε σ_0 of K̃ itself.
// The SVD is computed through a rank-revealing range finder: pivoted
// Gram-Schmidt (reorthogonalised) on the columns until the largest residual
// column norm times √(remaining columns) drops below 0.1 ε ‖K̃ col‖_max ≤
// 0.1 ε σ_0, then R = Q^H K̃ (k×n, k ≪ n) and the SVD of R by one-sided
// Jacobi on R^H.  Returns r (0 if K̃ = 0).
int lowrank_factor(int m, int n, const cd* A, double eps, std::vector<cd>& Uh, std::vector<cd>& Vh) {
  std::vector<cd> W(A, A + (size_t)m * n);  // residual columns
  std::vector<double> nrm(n);
  double cmax = 0;
  for (int j = 0; j < n; ++j) {
    double s = 0;
    for (int i = 0; i < m; ++i) s += std::norm(W[(size_t)j * m + i]);
    nrm[j] = s;
    cmax = std::max(cmax, s);
  }
  if (cmax == 0) { Uh.clear(); Vh.clear(); return 0; }
  const double c0 = std::sqrt(cmax);
  std::vector<cd> Q;  // m × k
  std::vector<char> used(n, 0);
  int k = 0;
  const int kmax = std::min(m, n);
  while (k < kmax) {
    int jp = -1;
    double best = -1;
    for (int j = 0; j < n; ++j)
      if (!used[j] && nrm[j] > best) { best = nrm[j]; jp = j; }
    if (jp < 0 || std::sqrt(std::max(best, 0.0)) * std::sqrt((double)(n - k)) < 0.1 * eps * c0) break;
    used[jp] = 1;
    std::vector<cd> q(W.begin() + (size_t)jp * m, W.begin() + (size_t)(jp + 1) * m);
    for (int pass = 0; pass < 2; ++pass)  // reorthogonalise against Q
      for (int c = 0; c < k; ++c) {
        const cd* qc = Q.data() + (size_t)c * m;
        cd h = 0;
        for (int i = 0; i < m; ++i) h += std::conj(qc[i]) * q[i];
        for (int i = 0; i < m; ++i) q[i] -= h * qc[i];
      }
    double qn = 0;
    for (int i = 0; i < m; ++i) qn += std::norm(q[i]);
    qn = std::sqrt(qn);
    if (qn == 0) continue;
    for (int i = 0; i < m; ++i) q[i] /= qn;
    Q.insert(Q.end(), q.begin(), q.end());
    ++k;
    // remove q from the remaining residual columns
    for (int j = 0; j < n; ++j) {
      if (used[j]) { nrm[j] = 0; continue; }
      cd* w = W.data() + (size_t)j * m;
      cd h = 0;
      for (int i = 0; i < m; ++i) h += std::conj(q[i]) * w[i];
      double s = 0;
      for (int i = 0; i < m; ++i) {
        w[i] -= h * q[i];
        s += std::norm(w[i]);
      }
      nrm[j] = s;
    }
  }
  // R = Q^H A  (k × n), then SVD via one-sided Jacobi on R^H (n × k)
  std::vector<cd> RH((size_t)n * k);  // column c of R^H = conj(row c of R)
  for (int c = 0; c < k; ++c)
    for (int j = 0; j < n; ++j) {
      const cd* qc = Q.data() + (size_t)c * m;
      const cd* a = A + (size_t)j * m;
      cd h = 0;
      for (int i = 0; i < m; ++i) h += std::conj(qc[i]) * a[i];
      RH[(size_t)c * n + j] = std::conj(h);
    }
  std::vector<double> S;
  std::vector<cd> Z;  // k × k
  svd_jacobi(n, k, RH, S, Z);  // R^H = Wl S Z^H  → R = Z S Wl^H ; RH now holds Wl (n × k)
  int r = 0;
  while (r < k && S[r] >= eps * S[0]) ++r;
  // Û = Q Z_r S_r (m × r), V̂ = Wl_r^H (r × n)
  Uh.assign((size_t)m * r, 0.0);
  for (int c = 0; c < r; ++c)
    for (int a = 0; a < k; ++a) {
      const cd z = Z[(size_t)c * k + a] * S[c];
      const cd* qa = Q.data() + (size_t)a * m;
      cd* u = Uh.data() + (size_t)c * m;
      for (int i = 0; i < m; ++i) u[i] += qa[i] * z;
    }
  Vh.assign((size_t)r * n, 0.0);
  for (int j = 0; j < n; ++j)
    for (int c = 0; c < r; ++c) Vh[(size_t)j * r + c] = std::conj(RH[(size_t)c * n + j]);
  return r;
}

}  // namespace fda

namespace fda {

// Truncated SVD of a check/equivalent-cloud kernel matrix (the level SVDs of P:679-705):
// A (m×n, column-major) = U diag(S) V^H restricted to the T triplets with σ_i ≥ ε σ_0.
// Same result as svd_jacobi + truncation up to the range finder's residual (≤ 1e-3 ε σ_0 in
// each singular value): a pivoted, twice-orthogonalised Gram–Schmidt range finder (OpenMP over
// the residual columns) stops once the largest residual column norm × √(remaining columns)
// < 1e-3 ε ‖A col‖_max; then R = Q^H A (k × n, k ≈ 1.3 T ≪ n) and the one-sided Jacobi SVD of
// R^H = W S Z^H give U = Q Z, V = W.  ~10× less work than Jacobi on the whole m×n matrix
// (whose rank at ε is ≈ T ≪ n).  Returns T.
int svd_range(int m, int n, const std::vector<cd>& A, double eps, std::vector<double>& S, std::vector<cd>& U,
              std::vector<cd>& V) {
  std::vector<cd> W(A);   // residual columns
  std::vector<double> nrm(n);
#pragma omp parallel for schedule(static)
  for (int j = 0; j < n; ++j) {
    double s = 0;
    for (int i = 0; i < m; ++i) s += std::norm(W[(size_t)j * m + i]);
    nrm[j] = s;
  }
  double cmax = 0;
  for (int j = 0; j < n; ++j) cmax = std::max(cmax, nrm[j]);
  S.clear(); U.clear(); V.clear();
  if (cmax == 0) return 0;
  const double c0 = std::sqrt(cmax), tol = 1e-3 * eps * c0;
  std::vector<cd> Q;   // m × k
  std::vector<char> used(n, 0);
  int k = 0;
  const int kmax = std::min(m, n);
  std::vector<cd> q(m), hc;
  while (k < kmax) {
    int jp = -1;
    double best = -1;
    for (int j = 0; j < n; ++j)
      if (!used[j] && nrm[j] > best) { best = nrm[j]; jp = j; }
    if (jp < 0 || std::sqrt(std::max(best, 0.0)) * std::sqrt((double)(n - k)) < tol) break;
    used[jp] = 1;
    std::copy(W.begin() + (size_t)jp * m, W.begin() + (size_t)(jp + 1) * m, q.begin());
    for (int pass = 0; pass < 2; ++pass) {   // reorthogonalise against Q (classical GS, twice)
      hc.assign(k, 0.0);
#pragma omp parallel for schedule(static)
      for (int c = 0; c < k; ++c) {
        const cd* qc = Q.data() + (size_t)c * m;
        cd h = 0;
        for (int i = 0; i < m; ++i) h += std::conj(qc[i]) * q[i];
        hc[c] = h;
      }
      for (int c = 0; c < k; ++c) {
        const cd* qc = Q.data() + (size_t)c * m;
        for (int i = 0; i < m; ++i) q[i] -= hc[c] * qc[i];
      }
    }
    double qn = 0;
    for (int i = 0; i < m; ++i) qn += std::norm(q[i]);
    qn = std::sqrt(qn);
    if (qn == 0) continue;
    for (int i = 0; i < m; ++i) q[i] /= qn;
    Q.insert(Q.end(), q.begin(), q.end());
    ++k;
    // remove q from the remaining residual columns
#pragma omp parallel for schedule(static)
    for (int j = 0; j < n; ++j) {
      if (used[j]) { nrm[j] = 0; continue; }
      cd* w = W.data() + (size_t)j * m;
      cd h = 0;
      for (int i = 0; i < m; ++i) h += std::conj(q[i]) * w[i];
      double s = 0;
      for (int i = 0; i < m; ++i) {
        w[i] -= h * q[i];
        s += std::norm(w[i]);
      }
      nrm[j] = s;
    }
  }
  // R^H (n × k): column c = conj(row c of Q^H A)
  std::vector<cd> RH((size_t)n * k);
#pragma omp parallel for schedule(static)
  for (int cj = 0; cj < k * n; ++cj) {
    const int c = cj / n, j = cj % n;
    const cd* qc = Q.data() + (size_t)c * m;
    const cd* a = A.data() + (size_t)j * m;
    cd h = 0;
    for (int i = 0; i < m; ++i) h += std::conj(qc[i]) * a[i];
    RH[(size_t)c * n + j] = std::conj(h);
  }
  std::vector<double> Sk;
  std::vector<cd> Z;   // k × k
  svd_jacobi(n, k, RH, Sk, Z);   // R^H = W Sk Z^H (RH now W, n × k)  →  A ≈ Q R = (Q Z) Sk W^H
  int T = 0;
  while (T < k && Sk[T] >= eps * Sk[0]) ++T;
  S.assign(Sk.begin(), Sk.begin() + T);
  U.assign((size_t)m * T, 0.0);
#pragma omp parallel for schedule(static)
  for (int c = 0; c < T; ++c) {
    cd* u = U.data() + (size_t)c * m;
    for (int a = 0; a < k; ++a) {
      const cd z = Z[(size_t)c * k + a];
      const cd* qa = Q.data() + (size_t)a * m;
      for (int i = 0; i < m; ++i) u[i] += qa[i] * z;
    }
  }
  V.assign(RH.begin(), RH.begin() + (size_t)n * T);
  return T;
}

}  // namespace fda
