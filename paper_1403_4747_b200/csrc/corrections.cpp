// Near-field correction tables C (LHS) and C_rhs (RHS operator, kind 1)
// (fp64 → complex64 CSR in tree order).
//
// The device applies the 3-point rule Q3 to every element pair, either on the
// fly (direct leaf pairs, near kernel) or folded into S2M (far pairs).  The
// operator of Eq. (5) with the tier rule of reading C6 differs
// from that only for pairs with ρ_ij = |x_i - c_j|/h_j < tier2_rho, so
//   C_ij = A^tier_ij - A^Q3_ij   (ρ_ij < 3, including i = j)
// where A^tier_ii = ½ + α H_ii (closed-form self term, reading C5) and the
// Q3 value of the self pair is the (regular) 3-point sum on Δ_i.  The pair
// search is a tree-independent radius search (one hash grid per element-size
// class) on the host;
// the entries are evaluated here (host build) or by build_dev.cu (device build,
// the same definitions in fp64 on the GPU).
#include <algorithm>
#include <parallel/algorithm>
#include <cmath>
#include <omp.h>

#include "fda_internal.h"

namespace fda {

void correction_pairs(const Geometry& g, const Params& p, std::vector<int64_t>& ptr, std::vector<int64_t>& col,
                      std::vector<int8_t>& tier, int64_t row0, int64_t row1) {
  // Size classes: source element j with h_j ∈ (h₀/2^{c+1}, h₀/2^c] (h₀ = max h) goes to class c, whose
  // hash grid has cells of t2·h₀/2^c.  A pair with ρ_ij < t2 has |x_i - c_j| < t2·h_j ≤ the class's cell,
  // so target i lies in one of the 27 cells around c_j's cell of j's class.  One grid per class keeps
  // the candidate count per pair bounded on graded meshes (config 4: h varies 8× along the spheroid;
  // a single grid sized for the largest element scanned ~60× more candidates at the tips).
  // Per non-empty source cell, the 27 neighbouring TARGET cells of the same grid (targets hashed into it,
  // sorted by key) are found by binary search; the (target cell, source cell) adjacency is then walked
  // target-cell major in two passes (count, fill) and each row sorted by column.
  const int64_t n = g.n;
  const double t1 = p.opt.tier1_rho, t2 = p.opt.tier2_rho;
  constexpr int NC = 12;
  double h0 = 0;
  Vec3 lo(1e300, 1e300, 1e300);
  for (int64_t i = 0; i < n; ++i) {
    h0 = std::max(h0, g.hmax[i]);
    lo = {std::min(lo.x, g.centroid[i].x), std::min(lo.y, g.centroid[i].y), std::min(lo.z, g.centroid[i].z)};
  }
  std::vector<int8_t> cls(n);
  int ncls = 0;
#pragma omp parallel for schedule(static) reduction(max : ncls)
  for (int64_t j = 0; j < n; ++j) {
    const int c = std::min(NC - 1, std::max(0, (int)std::floor(std::log2(h0 / g.hmax[j]))));
    cls[j] = (int8_t)c;
    ncls = std::max(ncls, c + 1);
  }
  auto hkey = [](int64_t a, int64_t b, int64_t d) {
    return (uint64_t)((a & 0x1fffff) | ((b & 0x1fffff) << 21) | ((d & 0x1fffff) << 42));
  };
  ptr.assign(n + 1, 0);
  std::vector<int64_t> cur(n + 1, 0);   // pass 0: counts; pass 1: fill cursors
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      for (int64_t i = 0; i < n; ++i) ptr[i + 1] = ptr[i] + cur[i];
      col.resize(ptr[n]);
      tier.resize(ptr[n]);
      std::copy(ptr.begin(), ptr.end() - 1, cur.begin());
    }
    for (int c = 0; c < ncls; ++c) {
      // the class's cell size: an upper bound of t2·h_j for its members (c = NC-1 takes every smaller h)
      const double cell = t2 * h0 * std::ldexp(1.0, -c);
      auto key_of = [&](const Vec3& v) {
        return hkey((int64_t)std::floor((v.x - lo.x) / cell), (int64_t)std::floor((v.y - lo.y) / cell),
                    (int64_t)std::floor((v.z - lo.z) / cell));
      };
      std::vector<std::pair<uint64_t, int64_t>> se, te;   // (cell key, element): sources of class c, own targets
      for (int64_t j = 0; j < n; ++j)
        if (cls[j] == c) se.push_back({0, j});
      if (se.empty()) continue;
#pragma omp parallel for schedule(static)
      for (int64_t q = 0; q < (int64_t)se.size(); ++q) se[q].first = key_of(g.centroid[se[q].second]);
      te.resize(row1 - row0);
#pragma omp parallel for schedule(static)
      for (int64_t i = row0; i < row1; ++i) te[i - row0] = {key_of(g.centroid[i]), i};
      __gnu_parallel::sort(se.begin(), se.end());
      __gnu_parallel::sort(te.begin(), te.end());
      std::vector<int64_t> sc, tc;   // starts of the source cells / target cells (runs of equal keys)
      for (int64_t q = 0; q < (int64_t)se.size(); ++q)
        if (q == 0 || se[q].first != se[q - 1].first) sc.push_back(q);
      sc.push_back((int64_t)se.size());
      for (int64_t q = 0; q < (int64_t)te.size(); ++q)
        if (q == 0 || te[q].first != te[q - 1].first) tc.push_back(q);
      tc.push_back((int64_t)te.size());
      const int64_t nsc = (int64_t)sc.size() - 1, ntc = (int64_t)tc.size() - 1;
      // adjacency (target cell, source cell) for every source cell and its 27 neighbours that hold targets,
      // sorted by target cell: each target cell is then processed by one thread and its rows are written
      // contiguously, without atomics
      std::vector<std::vector<uint64_t>> adj_t(omp_get_max_threads());
#pragma omp parallel
      {
        auto& out = adj_t[omp_get_thread_num()];
#pragma omp for schedule(static)
        for (int64_t s = 0; s < nsc; ++s) {
          const uint64_t k = se[sc[s]].first;
          const int64_t a = (int64_t)(k & 0x1fffff), b = (int64_t)((k >> 21) & 0x1fffff), d = (int64_t)(k >> 42);
          for (int64_t da = -1; da <= 1; ++da)
            for (int64_t db = -1; db <= 1; ++db)
              for (int64_t dd = -1; dd <= 1; ++dd) {
                const uint64_t nk = hkey(a + da, b + db, d + dd);
                int64_t lo_ = 0, hi_ = ntc;   // first target cell with key >= nk
                while (lo_ < hi_) {
                  const int64_t m = (lo_ + hi_) >> 1;
                  if (te[tc[m]].first < nk) lo_ = m + 1; else hi_ = m;
                }
                if (lo_ < ntc && te[tc[lo_]].first == nk) out.push_back(((uint64_t)lo_ << 32) | (uint64_t)s);
              }
        }
      }
      std::vector<uint64_t> adj;
      for (auto& v : adj_t) adj.insert(adj.end(), v.begin(), v.end());
      __gnu_parallel::sort(adj.begin(), adj.end());
      std::vector<int64_t> at;   // starts of each target cell's run in adj
      for (int64_t q = 0; q < (int64_t)adj.size(); ++q)
        if (q == 0 || (adj[q] >> 32) != (adj[q - 1] >> 32)) at.push_back(q);
      at.push_back((int64_t)adj.size());
      const int64_t nat = (int64_t)at.size() - 1;
#pragma omp parallel for schedule(dynamic, 16)
      for (int64_t u = 0; u < nat; ++u) {
        const int64_t t = (int64_t)(adj[at[u]] >> 32);
        for (int64_t w = tc[t]; w < tc[t + 1]; ++w) {
          const int64_t i = te[w].second;
          const Vec3& x = g.centroid[i];
          int64_t e = cur[i];
          for (int64_t v = at[u]; v < at[u + 1]; ++v) {
            const int64_t s = (int64_t)(adj[v] & 0xffffffffu);
            for (int64_t q = sc[s]; q < sc[s + 1]; ++q) {
              const int64_t j = se[q].second;
              const Vec3 dv = x - g.centroid[j];
              const double r2 = dv.dot(dv), hr = t2 * g.hmax[j];
              if (r2 > hr * hr * (1 + 1e-9)) continue;   // clearly outside; the test below decides the rest
              const double rho = dv.norm() / g.hmax[j];
              if (!(rho < t2)) continue;
              if (pass == 1) {
                col[e] = j;
                tier[e] = (int8_t)(j == i ? 0 : (rho < t1 ? 1 : 2));
              }
              ++e;
            }
          }
          cur[i] = e;
        }
      }
    }
  }
  // rows in column order (the CSR the engine and the debug tables expect)
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = row0; i < row1; ++i) {
    const int64_t b = ptr[i], e = ptr[i + 1];
    std::vector<std::pair<int64_t, int8_t>> row(e - b);
    for (int64_t q = b; q < e; ++q) row[q - b] = {col[q], tier[q]};
    std::sort(row.begin(), row.end());
    for (int64_t q = b; q < e; ++q) {
      col[q] = row[q - b].first;
      tier[q] = row[q - b].second;
    }
  }
}

void build_corrections(const Geometry& g, const Params& p, Plan& plan, int kind) {
  auto& ptr = kind == 0 ? plan.corr_ptr : plan.corr_ptr_rhs;
  auto& col = kind == 0 ? plan.corr_col : plan.corr_col_rhs;
  auto& val = kind == 0 ? plan.corr_val : plan.corr_val_rhs;
  std::vector<int8_t> tier;
  correction_pairs(g, p, ptr, col, tier, plan.own_e0, plan.own_e1);
  const int64_t n = g.n;
  val.resize(ptr[n]);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t i = 0; i < n; ++i) {
    const Vec3& x = g.centroid[i];
    for (int64_t e = ptr[i]; e < ptr[i + 1]; ++e) {
      const int64_t j = col[e];
      cd q3 = entry_rule(3, x, g.normal[i], g.v0[j], g.v1[j], g.v2[j], g.normal[j], g.area[j], p.k, p.alpha, kind);
      cd exact;
      if (tier[e] == 0)
        exact = kind == 0 ? self_lhs(g.v0[i], g.v1[i], g.v2[i], p.k, p.alpha)
                          : self_rhs(g.v0[i], g.v1[i], g.v2[i], p.k, p.alpha);
      else exact = entry_rule(tier[e], x, g.normal[i], g.v0[j], g.v1[j], g.v2[j], g.normal[j], g.area[j], p.k,
                              p.alpha, kind);
      const cd c = exact - q3;
      val[e] = cf((float)c.real(), (float)c.imag());
    }
  }
}

}  // namespace fda
