// Build-time tool: the correction pair search of corrections.cpp (one hash grid per element-size class)
// against the single-grid search it replaced (kept here as the reference), on a mesh dumped by
// tools/pairs/run.sh.  Checks that the CSR (ptr, col, tier) is identical and times both.
//   g++ -O2 -fopenmp pairs_check.cpp -L../../paper_1403_4747_b200 -lfda -o pairs_check
#include <chrono>
#include <cstdio>
#include <parallel/algorithm>
#include <cmath>
#include <unordered_map>
#include "../../paper_1403_4747_b200/csrc/fda_internal.h"

namespace ref {
using namespace fda;
void correction_pairs_single_grid(const Geometry& g, const Params& p, std::vector<int64_t>& ptr, std::vector<int64_t>& col,
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

}  // namespace ref

int main(int argc, char** argv) {
  if (argc < 2) { fprintf(stderr, "usage: pairs_check mesh.bin\n"); return 2; }
  FILE* f = fopen(argv[1], "rb");
  int64_t nv, nt;
  if (fread(&nv, 8, 1, f) != 1 || fread(&nt, 8, 1, f) != 1) return 2;
  std::vector<double> V(3 * nv);
  std::vector<int32_t> F(3 * nt);
  if (fread(V.data(), 8, 3 * nv, f) != (size_t)(3 * nv) || fread(F.data(), 4, 3 * nt, f) != (size_t)(3 * nt)) return 2;
  fclose(f);
  fda::Geometry g;
  std::string err;
  if (fda::build_geometry(V.data(), nv, F.data(), nt, g, err) != FDA_OK) { fprintf(stderr, "%s\n", err.c_str()); return 1; }
  fda::Params p{};
  fda_options_default(&p.opt);
  using clk = std::chrono::steady_clock;
  std::vector<int64_t> p0, c0, p1, c1;
  std::vector<int8_t> t0, t1;
  auto a = clk::now();
  fda::correction_pairs(g, p, p1, c1, t1, 0, g.n);
  auto b = clk::now();
  ref::correction_pairs_single_grid(g, p, p0, c0, t0, 0, g.n);
  auto c = clk::now();
  const bool same = p0 == p1 && c0 == c1 && t0 == t1;
  // a sharded row range too
  std::vector<int64_t> p2, c2, p3, c3;
  std::vector<int8_t> t2, t3;
  fda::correction_pairs(g, p, p2, c2, t2, g.n / 3, g.n / 2);
  ref::correction_pairs_single_grid(g, p, p3, c3, t3, g.n / 3, g.n / 2);
  const bool same_shard = p2 == p3 && c2 == c3 && t2 == t3;
  printf("{\"N\": %lld, \"entries\": %lld, \"class_grids_s\": %.3f, \"single_grid_s\": %.3f, \"identical\": %s, "
         "\"identical_row_range\": %s}\n",
         (long long)g.n, (long long)p1.back(), std::chrono::duration<double>(b - a).count(),
         std::chrono::duration<double>(c - b).count(), same ? "true" : "false", same_shard ? "true" : "false");
  return same && same_shard ? 0 : 1;
}
