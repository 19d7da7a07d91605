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
// search is a tree-independent radius search (uniform hash grid) on the host;
// the entries are evaluated here (host build) or by build_dev.cu (device build,
// the same definitions in fp64 on the GPU).
#include <algorithm>
#include <parallel/algorithm>
#include <cmath>
#include <unordered_map>

#include "fda_internal.h"

namespace fda {

void correction_pairs(const Geometry& g, const Params& p, std::vector<int64_t>& ptr, std::vector<int64_t>& col,
                      std::vector<int8_t>& tier, int64_t row0, int64_t row1) {
  const int64_t n = g.n;
  const double t1 = p.opt.tier1_rho, t2 = p.opt.tier2_rho;
  double hmax = 0;
  for (int64_t i = 0; i < n; ++i) hmax = std::max(hmax, g.hmax[i]);
  const double cell = t2 * hmax;
  Vec3 lo(1e300, 1e300, 1e300);
  for (int64_t i = 0; i < n; ++i)
    lo = {std::min(lo.x, g.centroid[i].x), std::min(lo.y, g.centroid[i].y), std::min(lo.z, g.centroid[i].z)};
  auto cidx = [&](const Vec3& c, int64_t& a, int64_t& b, int64_t& d) {
    a = (int64_t)std::floor((c.x - lo.x) / cell);
    b = (int64_t)std::floor((c.y - lo.y) / cell);
    d = (int64_t)std::floor((c.z - lo.z) / cell);
  };
  auto hkey = [](int64_t a, int64_t b, int64_t d) {
    return (uint64_t)((a & 0x1fffff) | ((b & 0x1fffff) << 21) | ((d & 0x1fffff) << 42));
  };
  // uniform grid: elements sorted by cell key (parallel sort), cell → [begin, end) in that order
  std::vector<std::pair<uint64_t, int64_t>> ce(n);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    int64_t a, b, d;
    cidx(g.centroid[j], a, b, d);
    ce[j] = {hkey(a, b, d), j};
  }
  __gnu_parallel::sort(ce.begin(), ce.end());
  std::unordered_map<uint64_t, std::pair<int64_t, int64_t>> grid;
  for (int64_t q = 0; q < n;) {
    int64_t r = q;
    while (r < n && ce[r].first == ce[q].first) ++r;
    grid.emplace(ce[q].first, std::make_pair(q, r));
    q = r;
  }
  // two passes over the rows: count, then fill the CSR in place (no per-row vectors)
  auto scan = [&](int64_t i, auto&& emit) {
    const Vec3& x = g.centroid[i];
    int64_t a, b, d;
    cidx(x, a, b, d);
    for (int64_t da = -1; da <= 1; ++da)
      for (int64_t db = -1; db <= 1; ++db)
        for (int64_t dd = -1; dd <= 1; ++dd) {
          auto it = grid.find(hkey(a + da, b + db, d + dd));
          if (it == grid.end()) continue;
          for (int64_t q = it->second.first; q < it->second.second; ++q) {
            const int64_t j = ce[q].second;
            const double rho = (x - g.centroid[j]).norm() / g.hmax[j];
            if (!(rho < t2)) continue;
            emit(j, (int8_t)(j == i ? 0 : (rho < t1 ? 1 : 2)));
          }
        }
  };
  ptr.assign(n + 1, 0);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i) {
    if (i < row0 || i >= row1) continue;   // another rank's row (sharded build)
    int64_t c = 0;
    scan(i, [&](int64_t, int8_t) { ++c; });
    ptr[i + 1] = c;
  }
  for (int64_t i = 0; i < n; ++i) ptr[i + 1] += ptr[i];
  col.resize(ptr[n]);
  tier.resize(ptr[n]);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i) {
    if (i < row0 || i >= row1) continue;
    std::vector<std::pair<int64_t, int8_t>> row;
    row.reserve(ptr[i + 1] - ptr[i]);
    scan(i, [&](int64_t j, int8_t tr) { row.push_back({j, tr}); });
    std::sort(row.begin(), row.end(), [](const auto& u, const auto& v) { return u.first < v.first; });
    for (size_t e = 0; e < row.size(); ++e) {
      col[ptr[i] + e] = row[e].first;
      tier[ptr[i] + e] = row[e].second;
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
