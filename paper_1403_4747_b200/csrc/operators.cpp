// Equivalent / check clouds, truncated SVDs and the compressed translation
// tables (host, fp64 → complex64).
//
// PAPER.md §3.1 and §4.1.2-§4.3:
//   G_up = G(OUT_CHECK, OUT_EQUIV) = U Σ V^H, truncated at σ_i < ε σ_0 (C15)
//   G_dn = G_up^T  (incoming clouds are the point reflection of the outgoing
//                   ones, reading C12)  ⇒ U_dn = conj(V), V_dn = conj(U)
//   S̃ = Σ̃⁻¹ Ũ^H E_up   T × n_B   per leaf
//   M̃ = Σ̃_l⁻¹ Ũ_l^H E_up Ṽ_{l+1}  per (level, octant, direction)
//   K̃ = Ũ_dn^H K Ṽ_up          (Eq. eq_cmpm2l) per (level, rotated offset)
//   L̃ = Ũ_dn,l+1^H E_dn Ṽ_dn,l Σ̃_l⁻¹
//   T̃ = E_dn Ṽ_dn Σ̃⁻¹   n_B × T   per leaf
// Clouds (readings C12-C14): OUT_EQUIV = cube grid (p_eq per edge, side
// 1.05 w); LF OUT_CHECK = cube grid (p_chk_lf, side 2.95 w); HF OUT_CHECK = the
// p_chk_hf cube grid mapped onto a +z frustum, ρ(c) = d_min (d_max/d_min)^{(c+1)/2},
// half-width ρ tan θ_w + (√3/2) w, θ_w = atan(√2/n_f), d_min = max(2w, w²/λ),
// d_max = root diagonal; the cloud of direction u is the reference cloud
// rotated by R_u^T (rotation invariance).
#include <algorithm>
#include <cmath>

#include "fda_internal.h"

namespace fda {

static std::vector<Vec3> cube_grid(int p, double side) {
  std::vector<Vec3> pts;
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      for (int k = 0; k < p; ++k) {
        bool surf = i == 0 || j == 0 || k == 0 || i == p - 1 || j == p - 1 || k == p - 1;
        if (!surf) continue;
        auto c = [&](int t) { return -0.5 * side + side * t / (p - 1); };
        pts.push_back({c(i), c(j), c(k)});
      }
  return pts;
}

static std::vector<Vec3> frustum(int p, double w, double lambda, int nf, double root_width) {
  std::vector<Vec3> pts;
  double dmin = std::max(2.0 * w, w * w / lambda);
  double dmax = std::max(std::sqrt(3.0) * root_width, 2.0 * dmin);
  double tanth = std::sqrt(2.0) / nf;
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j)
      for (int k = 0; k < p; ++k) {
        bool surf = i == 0 || j == 0 || k == 0 || i == p - 1 || j == p - 1 || k == p - 1;
        if (!surf) continue;
        double a = -1.0 + 2.0 * i / (p - 1), b = -1.0 + 2.0 * j / (p - 1), c = -1.0 + 2.0 * k / (p - 1);
        double rho = dmin * std::pow(dmax / dmin, 0.5 * (c + 1.0));
        double hw = rho * tanth + 0.5 * std::sqrt(3.0) * w;
        pts.push_back({a * hw, b * hw, rho});
      }
  return pts;
}

void build_clouds_and_svd(const Params& p, Tree& t, const std::vector<bool>& need) {
  for (size_t l = 0; l < t.levels.size(); ++l) {
    Level& L = t.levels[l];
    if (!need[l]) { L.rank = 0; continue; }
    L.eq = cube_grid(p.opt.p_eq, p.opt.eq_scale * L.width);
    if (L.hf) L.chk = frustum(p.opt.p_chk_hf, L.width, t.lambda, L.nf, t.root_width);
    else L.chk = cube_grid(p.opt.p_chk_lf, p.opt.chk_scale_lf * L.width);
    const int m = (int)L.chk.size(), n = (int)L.eq.size();
    std::vector<cd> A((size_t)m * n);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < m; ++i) A[(size_t)j * m + i] = G(L.chk[i], L.eq[j], p.k);
    L.rank = svd_range(m, n, A, p.eps, L.S, L.U, L.V);   // σ_i ≥ ε σ_0
  }
}

// frame rotation of an out-state (dir u) or in-state (dir w: frame of anti(w))
Mat3 out_frame(const Level& L, int dir) {
  if (dir < 0) return rotation_to_z(Vec3(0, 0, 1));
  return rotation_to_z(dir_center(dir, L.nf));
}
Mat3 in_frame(const Level& L, int dir) {
  if (dir < 0) return rotation_to_z(Vec3(0, 0, 1));
  return rotation_to_z(dir_center(anti_dir(dir, L.nf), L.nf));
}
Vec3 octant_offset(int o, double wc) {
  return Vec3(((o & 1) ? 0.5 : -0.5) * wc, ((o >> 1) & 1 ? 0.5 : -0.5) * wc, ((o >> 2) & 1 ? 0.5 : -0.5) * wc);
}

static void store(Plan& plan, int64_t id, int rows, int cols, const std::vector<cd>& M) {
  cf* dst = plan.pool.data() + plan.mats[id].offset;
  for (size_t i = 0; i < (size_t)rows * cols; ++i) dst[i] = cf((float)M[i].real(), (float)M[i].imag());
}

void operator_layout(const Tree& t, Plan& plan, const std::vector<char>& needed) {
  const int64_t nm = (int64_t)plan.specs.size();
  plan.mats.resize(nm);
  int64_t off = 0, lr_bound = 0;
  for (int64_t id = 0; id < nm; ++id) {
    const MatSpec& s = plan.specs[id];
    int rows = 0, cols = 0;
    switch (s.kind) {
      case MK_S2M:
      case MK_S2M_RHS: {
        const Box& B = t.boxes[s.leaf];
        rows = t.levels[s.level].rank; cols = (int)(B.end - B.begin);
      } break;
      case MK_L2T: {
        const Box& B = t.boxes[s.leaf];
        rows = (int)(B.end - B.begin); cols = t.levels[s.level].rank;
      } break;
      case MK_M2M: rows = t.levels[s.level].rank; cols = t.levels[s.level + 1].rank; break;
      case MK_L2L: rows = t.levels[s.level + 1].rank; cols = t.levels[s.level].rank; break;
      case MK_M2L: rows = cols = t.levels[s.level].rank; break;
    }
    if (!needed.empty() && !needed[id]) rows = cols = 0;   // another rank's matrix (sharded build)
    plan.mats[id] = {off, rows, cols};
    off += (int64_t)rows * cols;
    if (s.kind == MK_M2L) lr_bound += (int64_t)rows * cols;   // §4.2 factors: 2·r·T < T² entries
  }
  plan.pool.clear();
  plan.pool.reserve(off + lr_bound);   // the factors are appended without reallocating
  plan.pool.resize(off);               // (uninitialised: every stored matrix is written in full)
}

// §4.2: K̃ ≈ Û V̂ of one T × T M2L matrix, kept when r < T/2
void lowrank_one(const Params& p, int64_t id, int T, const cd* M, LowRank& lr) {
  std::vector<cd> Uh, Vh;
  const int r = lowrank_factor(T, T, M, p.eps, Uh, Vh);
  if (r > 0 && 2 * r < T) {
    lr.R[id] = r;
    lr.U[id].swap(Uh);
    lr.V[id].swap(Vh);
  }
}

// every spec not already computed on the device (done[id] = 1), then the §4.2 factors
void build_operators(const Geometry& g, const Params& p, Tree& t, Plan& plan, const std::vector<char>& done,
                     LowRank& lr) {
  const int64_t nm = (int64_t)plan.specs.size();
  if ((int64_t)lr.R.size() != nm) { lr.R.assign(nm, -1); lr.U.assign(nm, {}); lr.V.assign(nm, {}); }
  std::vector<int>& lrR = lr.R;
  std::vector<std::vector<cd>>& lrU = lr.U;
  std::vector<std::vector<cd>>& lrV = lr.V;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t id = 0; id < nm; ++id) {
    if (!done.empty() && done[id]) continue;
    if (plan.mats[id].rows == 0) continue;   // not needed on this rank
    const MatSpec& s = plan.specs[id];
    const Level& L = t.levels[s.level];
    const int m = (int)L.chk.size(), n = (int)L.eq.size(), T = L.rank;
    std::vector<cd> E, X, M;
    switch (s.kind) {
      case MK_S2M:
      case MK_S2M_RHS: {
        // E_up[c, j] = Σ_q (A_j/3) ∂G/∂n_y(chk_c, y_jq)   (Eq. 10);
        // the RHS pass uses G sources
        const Box& B = t.boxes[s.leaf];
        const int nb = (int)(B.end - B.begin);
        E.resize((size_t)m * nb);
        // HF leaf (s.dir ≥ 0): the check cloud of wedge u, R_u^T chk (as for M2M)
        const Mat3 Rs = out_frame(L, s.dir);
        for (int j = 0; j < nb; ++j) {
          const int64_t e = B.begin + j;
          for (int c = 0; c < m; ++c) {
            Vec3 xc = B.center + (s.dir >= 0 ? Rs.apply_t(L.chk[c]) : L.chk[c]);
            cd acc = 0.0;
            for (int q = 0; q < 3; ++q) {
              Vec3 y = g.v0[e] * Q3_BARY[q][0] + g.v1[e] * Q3_BARY[q][1] + g.v2[e] * Q3_BARY[q][2];
              acc += s.kind == MK_S2M ? dGdny(xc, y, g.normal[e], p.k) : G(xc, y, p.k);
            }
            E[(size_t)j * m + c] = acc * (g.area[e] / 3.0);
          }
        }
        M.resize((size_t)T * nb);
        zgemm_cm(T, nb, m, L.U.data(), m, E.data(), m, M.data(), T, true);
        for (int j = 0; j < nb; ++j)
          for (int r = 0; r < T; ++r) M[(size_t)j * T + r] /= L.S[r];
        store(plan, id, T, nb, M);
      } break;
      case MK_L2T: {
        // E_dn[i, j] = G(x_i, y_j) + α ∂G/∂n_x(x_i, y_j), y_j = IN_EQUIV = c_B - chk_j  (Eq. 12)
        const Box& B = t.boxes[s.leaf];
        const int nb = (int)(B.end - B.begin);
        E.resize((size_t)nb * m);
        // HF leaf (s.dir = incoming wedge w ≥ 0): IN_EQUIV of w, R^T (−chk) in the frame of anti(w) (as for L2L)
        const Mat3 Qs = in_frame(L, s.dir);
        for (int j = 0; j < m; ++j) {
          Vec3 y = B.center + (s.dir >= 0 ? Qs.apply_t(-L.chk[j]) : -L.chk[j]);
          for (int i = 0; i < nb; ++i) {
            const int64_t e = B.begin + i;
            E[(size_t)j * nb + i] = G(g.centroid[e], y, p.k) + p.alpha * dGdnx(g.centroid[e], g.normal[e], y, p.k);
          }
        }
        // T̃ = E_dn conj(U) Σ̃⁻¹
        std::vector<cd> Uc(L.U.size());
        for (size_t i = 0; i < Uc.size(); ++i) Uc[i] = std::conj(L.U[i]);
        M.resize((size_t)nb * T);
        zgemm_cm(nb, T, m, E.data(), nb, Uc.data(), m, M.data(), nb, false);
        for (int c = 0; c < T; ++c)
          for (int i = 0; i < nb; ++i) M[(size_t)c * nb + i] /= L.S[c];
        store(plan, id, nb, T, M);
      } break;
      case MK_M2M: {
        const Level& Lc = t.levels[s.level + 1];
        const int nc = (int)Lc.eq.size(), Tc = Lc.rank;
        Mat3 Rp = out_frame(L, s.dir);
        int cdir = (Lc.hf && s.dir >= 0) ? child_dir(s.dir, L.nf) : -1;
        Mat3 Rc = out_frame(Lc, cdir);
        Vec3 oc = octant_offset(s.octant, Lc.width);
        E.resize((size_t)m * nc);
        for (int j = 0; j < nc; ++j) {
          Vec3 y = oc + Rc.apply_t(Lc.eq[j]);
          for (int i = 0; i < m; ++i) E[(size_t)j * m + i] = G(Rp.apply_t(L.chk[i]), y, p.k);
        }
        X.resize((size_t)m * Tc);
        zgemm_cm(m, Tc, nc, E.data(), m, Lc.V.data(), nc, X.data(), m, false);
        M.resize((size_t)T * Tc);
        zgemm_cm(T, Tc, m, L.U.data(), m, X.data(), m, M.data(), T, true);
        for (int j = 0; j < Tc; ++j)
          for (int r = 0; r < T; ++r) M[(size_t)j * T + r] /= L.S[r];
        store(plan, id, T, Tc, M);
      } break;
      case MK_L2L: {
        const Level& Lc = t.levels[s.level + 1];
        const int nc = (int)Lc.eq.size(), Tc = Lc.rank;
        Mat3 Qp = in_frame(L, s.dir);
        int cdir = (Lc.hf && s.dir >= 0) ? child_dir(s.dir, L.nf) : -1;
        Mat3 Qc = in_frame(Lc, cdir);
        Vec3 oc = octant_offset(s.octant, Lc.width);
        // E_dn[i, j] = G(child IN_CHECK_i, parent IN_EQUIV_j)
        E.resize((size_t)nc * m);
        for (int j = 0; j < m; ++j) {
          Vec3 y = Qp.apply_t(-L.chk[j]);
          for (int i = 0; i < nc; ++i) E[(size_t)j * nc + i] = G(oc + Qc.apply_t(-Lc.eq[i]), y, p.k);
        }
        std::vector<cd> Uc(L.U.size());
        for (size_t i = 0; i < Uc.size(); ++i) Uc[i] = std::conj(L.U[i]);
        X.resize((size_t)nc * T);
        zgemm_cm(nc, T, m, E.data(), nc, Uc.data(), m, X.data(), nc, false);
        for (int c = 0; c < T; ++c)
          for (int i = 0; i < nc; ++i) X[(size_t)c * nc + i] /= L.S[c];
        // L̃ = V_c^T X  = (conj V_c)^H X
        std::vector<cd> Vcc(Lc.V.size());
        for (size_t i = 0; i < Vcc.size(); ++i) Vcc[i] = std::conj(Lc.V[i]);
        M.resize((size_t)Tc * T);
        zgemm_cm(Tc, T, nc, Vcc.data(), nc, X.data(), nc, M.data(), Tc, true);
        store(plan, id, Tc, T, M);
      } break;
      case MK_M2L: {
        // K[i, j] = G(IN_CHECK(D)_i, OUT_EQUIV(C)_j) with both clouds in the frame R_u
        Mat3 R = out_frame(L, s.dir);
        Vec3 d((double)s.dx * L.width, (double)s.dy * L.width, (double)s.dz * L.width);
        E.resize((size_t)n * n);
        for (int j = 0; j < n; ++j) {
          Vec3 y = R.apply_t(L.eq[j]);
          for (int i = 0; i < n; ++i) E[(size_t)j * n + i] = G(d + R.apply_t(-L.eq[i]), y, p.k);
        }
        X.resize((size_t)n * T);
        zgemm_cm(n, T, n, E.data(), n, L.V.data(), n, X.data(), n, false);
        std::vector<cd> Vc(L.V.size());
        for (size_t i = 0; i < Vc.size(); ++i) Vc[i] = std::conj(L.V[i]);
        M.resize((size_t)T * T);
        zgemm_cm(T, T, n, Vc.data(), n, X.data(), n, M.data(), T, true);  // V^T (K V)
        store(plan, id, T, T, M);
        if (p.opt.m2l_lowrank) lowrank_one(p, id, T, M.data(), lr);
      } break;
    }
  }
  // append the §4.2 factors as new matrices: V̂ (r × T) then Û (T × r)
  plan.lr_V.assign(nm, -1);
  plan.lr_U.assign(nm, -1);
  int64_t off = (int64_t)plan.pool.size();
  std::vector<std::pair<int64_t, const std::vector<cd>*>> fill;   // (pool offset, factor)
  for (int64_t id = 0; id < nm; ++id) {
    if (lrR[id] < 0) continue;
    const int r = lrR[id], T = plan.mats[id].rows;
    for (int w = 0; w < 2; ++w) {
      const int64_t nid = (int64_t)plan.mats.size();
      MatInfo mi{off, w == 0 ? r : T, w == 0 ? T : r};
      plan.mats.push_back(mi);
      plan.specs.push_back(plan.specs[id]);
      fill.push_back({off, w == 0 ? &lrV[id] : &lrU[id]});
      off += (int64_t)r * T;
      (w == 0 ? plan.lr_V : plan.lr_U)[id] = nid;
    }
  }
  plan.pool.resize(off);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t f = 0; f < (int64_t)fill.size(); ++f) {
    const std::vector<cd>& src = *fill[f].second;
    cf* dst = plan.pool.data() + fill[f].first;
    for (size_t e = 0; e < src.size(); ++e) dst[e] = cf((float)src[e].real(), (float)src[e].imag());
  }
}

}  // namespace fda
