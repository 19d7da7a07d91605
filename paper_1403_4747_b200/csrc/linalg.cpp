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
