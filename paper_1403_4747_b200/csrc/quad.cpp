// fp64 kernels, triangle rules and singular self terms used by the build
// (near-field correction table and translation-operator generation).
//
// Kernels: G = e^{ikr}/(4πr) (Eq. 3).  With d = x - y, q = kr,
// a = d·n_x/r, b = -d·n_y/r, c = n_x·n_y and E = e^{iq}/(4πr²):
//   ∂G/∂n_y        = E (iq - 1) b
//   ∂G/∂n_x        = E (iq - 1) a
//   ∂²G/∂n_x∂n_y   = (E/r) [ (3 - q²) ab + c - i q (3ab + c) ]
// (the Burton–Miller LHS integrand of Eq. (5), is ∂G/∂n_y + α ∂²G/∂n_x∂n_y).
// Rules (reading C6): Q3 Strang-Fix (2/3,1/6,1/6); Q6 Dunavant degree 4;
// Q7 Radon degree 5; T1 = Q7 on the depth-3 1:4 subdivision (448 points).
// Self terms (reading C5): H_ii = FP∫ r⁻³/(4π) + ∫[e^{iq}(1-iq)-1]/(4πr³),
// static part in closed form per edge, remainder by polar Gauss-Legendre 20×20.
#include <cmath>
#include <array>
#include <vector>

#include "fda_internal.h"

namespace fda {

static const double kPi = 3.14159265358979323846;
const double Q3_BARY[3][3] = {{2.0 / 3, 1.0 / 6, 1.0 / 6}, {1.0 / 6, 2.0 / 3, 1.0 / 6}, {1.0 / 6, 1.0 / 6, 2.0 / 3}};

namespace {
struct Rules {
  double q6[6][3], w6[6];
  double q7[7][3], w7[7];
  double t1[448][3], wt1[448];
  double gl_x[20], gl_w[20];
  Rules() {
    auto orbit = [](double (*P)[3], double* W, int at, double a, double w) {
      double b = 1.0 - 2.0 * a;
      const double pts[3][3] = {{b, a, a}, {a, b, a}, {a, a, b}};
      for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) P[at + i][j] = pts[i][j];
        W[at + i] = w;
      }
    };
    orbit(q6, w6, 0, 0.445948490915965, 0.223381589678011);
    orbit(q6, w6, 3, 0.091576213509771, 0.109951743655322);
    const double r15 = std::sqrt(15.0);
    q7[0][0] = q7[0][1] = q7[0][2] = 1.0 / 3.0;
    w7[0] = 0.225;
    orbit(q7, w7, 1, (6.0 - r15) / 21.0, (155.0 - r15) / 1200.0);
    orbit(q7, w7, 4, (6.0 + r15) / 21.0, (155.0 + r15) / 1200.0);
    // depth-3 subdivision: iterate sub-triangles as barycentric corner triples
    std::vector<std::array<std::array<double, 3>, 3>> tris{{{{{1, 0, 0}}, {{0, 1, 0}}, {{0, 0, 1}}}}};
    for (int d = 0; d < 3; ++d) {
      std::vector<std::array<std::array<double, 3>, 3>> nx;
      for (auto& T : tris) {
        std::array<double, 3> ab, bc, ca;
        for (int c = 0; c < 3; ++c) {
          ab[c] = 0.5 * (T[0][c] + T[1][c]);
          bc[c] = 0.5 * (T[1][c] + T[2][c]);
          ca[c] = 0.5 * (T[2][c] + T[0][c]);
        }
        nx.push_back({T[0], ab, ca});
        nx.push_back({ab, T[1], bc});
        nx.push_back({ca, bc, T[2]});
        nx.push_back({ab, bc, ca});
      }
      tris.swap(nx);
    }
    int cnt = 0;
    for (auto& T : tris)
      for (int q = 0; q < 7; ++q) {
        for (int c = 0; c < 3; ++c) t1[cnt][c] = q7[q][0] * T[0][c] + q7[q][1] * T[1][c] + q7[q][2] * T[2][c];
        wt1[cnt] = w7[q] / 64.0;
        ++cnt;
      }
    // Gauss-Legendre 20 on [-1,1] by Newton on P_20
    const int n = 20;
    for (int i = 0; i < n; ++i) {
      double x = std::cos(kPi * (i + 0.75) / (n + 0.5));
      for (int it = 0; it < 100; ++it) {
        double p0 = 1.0, p1 = x;
        for (int k = 2; k <= n; ++k) {
          double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
          p0 = p1; p1 = p2;
        }
        double dp = n * (x * p1 - p0) / (x * x - 1.0);
        double dx = p1 / dp;
        x -= dx;
        if (std::fabs(dx) < 1e-16) break;
      }
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1; p1 = p2;
      }
      double dp = n * (x * p1 - p0) / (x * x - 1.0);
      gl_x[i] = x;
      gl_w[i] = 2.0 / ((1.0 - x * x) * dp * dp);
    }
  }
};
const Rules& rules() {
  static Rules r;
  return r;
}
}  // namespace

void quad_tables(std::vector<double>& t1, std::vector<double>& q6, std::vector<double>& gl) {
  const Rules& R = rules();
  t1.clear(); q6.clear(); gl.clear();
  for (int q = 0; q < 448; ++q) { t1.insert(t1.end(), {R.t1[q][0], R.t1[q][1], R.t1[q][2], R.wt1[q]}); }
  for (int q = 0; q < 6; ++q) { q6.insert(q6.end(), {R.q6[q][0], R.q6[q][1], R.q6[q][2], R.w6[q]}); }
  for (int i = 0; i < 20; ++i) { gl.push_back(R.gl_x[i]); gl.push_back(R.gl_w[i]); }
}

cd G(const Vec3& x, const Vec3& y, double k) {
  double r = (x - y).norm();
  return std::polar(1.0, k * r) / (4.0 * kPi * r);
}

cd dGdnx(const Vec3& x, const Vec3& nx, const Vec3& y, double k) {
  Vec3 d = x - y;
  double r = d.norm(), q = k * r;
  cd E = std::polar(1.0 / (4.0 * kPi * r * r), q);
  return E * cd(-1.0, q) * (d.dot(nx) / r);
}

cd dGdny(const Vec3& x, const Vec3& y, const Vec3& ny, double k) {
  Vec3 d = x - y;
  double r = d.norm(), q = k * r;
  cd E = std::polar(1.0 / (4.0 * kPi * r * r), q);
  return E * cd(-1.0, q) * (-d.dot(ny) / r);
}

cd lhs_kernel(const Vec3& x, const Vec3& nx, const Vec3& y, const Vec3& ny, double k, cd alpha) {
  Vec3 d = x - y;
  double r = d.norm(), q = k * r, ir = 1.0 / r;
  double a = d.dot(nx) * ir, b = -d.dot(ny) * ir, c = nx.dot(ny);
  cd E = std::polar(ir * ir / (4.0 * kPi), q);
  cd D = E * cd(-b, q * b);
  double ab = a * b;
  cd H = E * ir * cd((3.0 - q * q) * ab + c, -q * (3.0 * ab + c));
  return D + alpha * H;
}

// RHS integrand of Eq. (4): G + α ∂G/∂n_x = E [ r + α (iq - 1) a ]
cd rhs_kernel(const Vec3& x, const Vec3& nx, const Vec3& y, double k, cd alpha) {
  Vec3 d = x - y;
  double r = d.norm(), q = k * r, ir = 1.0 / r;
  double a = d.dot(nx) * ir;
  cd E = std::polar(ir * ir / (4.0 * kPi), q);
  return E * (r + alpha * cd(-a, q * a));
}

cd entry_rule(int tier, const Vec3& x, const Vec3& nx, const Vec3& A, const Vec3& B, const Vec3& C,
              const Vec3& ny, double area, double k, cd alpha, int kind) {
  const Rules& R = rules();
  const double(*P)[3];
  const double* W;
  int nq;
  static const double w3[3] = {1.0 / 3, 1.0 / 3, 1.0 / 3};
  if (tier == 3) { P = Q3_BARY; W = w3; nq = 3; }
  else if (tier == 2) { P = R.q6; W = R.w6; nq = 6; }
  else { P = R.t1; W = R.wt1; nq = 448; }
  cd s = 0.0;
  for (int q = 0; q < nq; ++q) {
    Vec3 y = A * P[q][0] + B * P[q][1] + C * P[q][2];
    s += W[q] * (kind == 0 ? lhs_kernel(x, nx, y, ny, k, alpha) : rhs_kernel(x, nx, y, k, alpha));
  }
  return area * s;
}

// ∫_Δ f dS with r·f(r) = g(r) smooth, polar GL 20×20 per edge sub-triangle
template <class Fn>
static cd polar_remainder(const Vec3 v[3], const Vec3& x, Fn g) {
  const Rules& R = rules();
  cd total = 0.0;
  for (int e = 0; e < 3; ++e) {
    Vec3 va = v[e], vb = v[(e + 1) % 3];
    Vec3 u = (vb - va) * (1.0 / (vb - va).norm());
    double ta = (va - x).dot(u), tb = (vb - x).dot(u);
    double dlt = ((va - x) - u * ta).norm();
    double pa = std::atan2(ta, dlt), pb = std::atan2(tb, dlt);
    for (int i = 0; i < 20; ++i) {
      double psi = 0.5 * (pb - pa) * R.gl_x[i] + 0.5 * (pb + pa);
      double wpsi = 0.5 * (pb - pa) * R.gl_w[i];
      double Rm = dlt / std::cos(psi);
      cd inner = 0.0;
      for (int j = 0; j < 20; ++j) {
        double rr = 0.5 * Rm * (R.gl_x[j] + 1.0);
        inner += (0.5 * Rm * R.gl_w[j]) * g(rr);
      }
      total += wpsi * inner;
    }
  }
  return total;
}

cd self_lhs(const Vec3& A, const Vec3& B, const Vec3& C, double k, cd alpha) {
  const Vec3 v[3] = {A, B, C};
  const Vec3 x = (A + B + C) * (1.0 / 3.0);
  double fp = 0.0;  // FP∫ r⁻³ = -Σ (t_b/ρ_b - t_a/ρ_a)/δ
  for (int e = 0; e < 3; ++e) {
    Vec3 va = v[e], vb = v[(e + 1) % 3];
    Vec3 u = (vb - va) * (1.0 / (vb - va).norm());
    double ta = (va - x).dot(u), tb = (vb - x).dot(u);
    double dlt = ((va - x) - u * ta).norm();
    fp -= (tb / (vb - x).norm() - ta / (va - x).norm()) / dlt;
  }
  cd rem = polar_remainder(v, x, [k](double r) {
    cd e = std::polar(1.0, k * r);
    return (e * cd(1.0, -k * r) - 1.0) / (4.0 * kPi * r * r);
  });
  cd H = fp / (4.0 * kPi) + rem;
  return 0.5 + alpha * H;   // c = ½, D_ii = 0 on a flat panel (C3-C5)
}

// RHS diagonal: B_ii = -α/2 + S_ii, S_ii = (1/4π)∫r⁻¹ + ∫(e^{ikr}-1)/(4πr), K'_ii = 0
// (C4-C5; ∫_Δ r⁻¹ = Σ_e δ_e ln[(t_b+ρ_b)/(t_a+ρ_a)], App. B)
cd self_rhs(const Vec3& A, const Vec3& B, const Vec3& C, double k, cd alpha) {
  const Vec3 v[3] = {A, B, C};
  const Vec3 x = (A + B + C) * (1.0 / 3.0);
  double r1 = 0.0;
  for (int e = 0; e < 3; ++e) {
    Vec3 va = v[e], vb = v[(e + 1) % 3];
    Vec3 u = (vb - va) * (1.0 / (vb - va).norm());
    double ta = (va - x).dot(u), tb = (vb - x).dot(u);
    double dlt = ((va - x) - u * ta).norm();
    r1 += dlt * std::log((tb + (vb - x).norm()) / (ta + (va - x).norm()));
  }
  cd rem = polar_remainder(v, x, [k](double r) { return (std::polar(1.0, k * r) - 1.0) / (4.0 * kPi); });
  cd S = r1 / (4.0 * kPi) + rem;
  return -0.5 * alpha + S;
}

}  // namespace fda
