// Adaptive octree, regimes, directional wedges and interaction lists (host).
//
// PAPER.md Algorithm Step 1: construct the octree adaptively,
// define far fields, split LF/HF regimes, divide the HF far fields into
// directional cones, build the interaction lists.  Readings:
//  C7  root = axis-aligned cube at the vertex-bbox centre, width = max
//      extent·(1+2⁻²⁰); split while a cube owns > max_leaf elements; elements
//      owned by centroid; Morton order of centroids = internal "tree order".
//  C8  HF ⇔ w ≥ λ = 2π/k.
//  C9  HF cubes are always split (all leaves are LF) — unless opt.hf_leaves,
//      the paper's rule: split while > max_leaf elements at every level (HF leaves).
//  C10 wedges: 6·4^j face-grid squares, j = ⌈log₂(w/λ)⌉; the wedge of v is
//      the square hit on its dominant face; ties → lowest index; child map =
//      face index >> 1.
//  C11 adm_l(B,C) ⇔ Chebyshev index distance ≥ 2 ∧ (LF ∨ ‖Δc‖ ≥ w²/λ);
//      IL_l(B) = {adm_l(B,C) ∧ ¬adm_{l-1}(parents)}; leaf pairs with
//      ¬adm at the coarser leaf's level are direct.
//  C18 R_u = minimal rotation taking the wedge centre u to +z; the incoming
//      state of D is keyed by the antipodal wedge of C's outgoing wedge.
#include <algorithm>
#include <parallel/algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <tuple>
#include <unordered_map>

#include "fda_internal.h"

namespace fda {

static const int kMortonBits = 21;

double Params::lambda() const { return 2.0 * M_PI / k; }

static uint64_t spread3(uint64_t v) {
  uint64_t x = v & 0x1fffff;
  x = (x | x << 32) & 0x1f00000000ffffULL;
  x = (x | x << 16) & 0x1f0000ff0000ffULL;
  x = (x | x << 8) & 0x100f00f00f00f00fULL;
  x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
  x = (x | x << 2) & 0x1249249249249249ULL;
  return x;
}

void build_tree(Geometry& g, const Params& p, Tree& t) {
  const int64_t n = g.n;
  Vec3 lo(1e300, 1e300, 1e300), hi(-1e300, -1e300, -1e300);
  auto upd = [&](const Vec3& q) {
    lo = {std::min(lo.x, q.x), std::min(lo.y, q.y), std::min(lo.z, q.z)};
    hi = {std::max(hi.x, q.x), std::max(hi.y, q.y), std::max(hi.z, q.z)};
  };
  for (int64_t i = 0; i < n; ++i) { upd(g.v0[i]); upd(g.v1[i]); upd(g.v2[i]); }
  t.lambda = p.lambda();
  t.root_center = (lo + hi) * 0.5;
  double ext = std::max({hi.x - lo.x, hi.y - lo.y, hi.z - lo.z});
  t.root_width = ext * (1.0 + std::ldexp(1.0, -20));
  const Vec3 corner = t.root_center - Vec3(1, 1, 1) * (0.5 * t.root_width);
  const double scale = std::ldexp(1.0, kMortonBits) / t.root_width;
  const int64_t maxc = (int64_t(1) << kMortonBits) - 1;

  std::vector<uint64_t> key(n);
  std::vector<int64_t> ix(n), iy(n), iz(n);
  for (int64_t i = 0; i < n; ++i) {
    Vec3 c = g.centroid[i] - corner;
    ix[i] = std::min<int64_t>(maxc, std::max<int64_t>(0, (int64_t)std::floor(c.x * scale)));
    iy[i] = std::min<int64_t>(maxc, std::max<int64_t>(0, (int64_t)std::floor(c.y * scale)));
    iz[i] = std::min<int64_t>(maxc, std::max<int64_t>(0, (int64_t)std::floor(c.z * scale)));
    key[i] = spread3(ix[i]) | (spread3(iy[i]) << 1) | (spread3(iz[i]) << 2);
  }
  std::vector<int64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  __gnu_parallel::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return key[a] < key[b]; });
  // permute geometry into tree order
  auto permute = [&](auto& vec) {
    auto tmp = vec;
    for (int64_t i = 0; i < n; ++i) vec[i] = tmp[order[i]];
  };
  permute(g.v0); permute(g.v1); permute(g.v2); permute(g.centroid); permute(g.normal);
  permute(g.area); permute(g.hmax); permute(g.perm); permute(key); permute(ix); permute(iy); permute(iz);

  const double lam = p.lambda();
  t.boxes.clear();
  t.levels.clear();
  Box root{};
  root.level = 0; root.ix = root.iy = root.iz = 0; root.center = t.root_center; root.parent = -1;
  for (auto& c : root.child) c = -1;
  root.begin = 0; root.end = n; root.leaf = true; root.octant = 0;
  t.boxes.push_back(root);
  int64_t lvl_begin = 0, lvl_end = 1;
  for (int l = 0;; ++l) {
    Level L;
    L.width = t.root_width / std::ldexp(1.0, l);
    L.hf = (L.width >= lam) && !p.opt.direct_all;
    L.nf = 0;
    if (L.hf) {
      int j = 0;
      while (lam * std::ldexp(1.0, j) < L.width) ++j;
      L.nf = 1 << j;
    }
    L.ndir = L.hf ? 6 * L.nf * L.nf : 0;
    L.box_begin = lvl_begin; L.box_end = lvl_end;
    t.levels.push_back(L);
    if (l + 1 >= kMortonBits) break;
    int64_t next_begin = (int64_t)t.boxes.size();
    const int shift = kMortonBits - 1 - l;  // bit giving the child octant at level l+1
    for (int64_t b = lvl_begin; b < lvl_end; ++b) {
      // copies, not a reference: t.boxes grows (and may reallocate) inside the loop
      const int64_t b_begin = t.boxes[b].begin, b_end = t.boxes[b].end;
      int64_t cnt = b_end - b_begin;
      bool split = (L.hf && !p.opt.hf_leaves) ? (cnt > 0) : (cnt > p.opt.max_leaf);   // C9 / P:344-346
      if (!split) continue;
      int64_t s = b_begin;
      for (int o = 0; o < 8; ++o) {
        int64_t e = s;
        while (e < b_end) {
          int oo = (int)(((ix[e] >> shift) & 1) | (((iy[e] >> shift) & 1) << 1) | (((iz[e] >> shift) & 1) << 2));
          if (oo != o) break;
          ++e;
        }
        if (e > s) {
          Box C{};
          C.level = l + 1;
          C.ix = 2 * t.boxes[b].ix + (o & 1);
          C.iy = 2 * t.boxes[b].iy + ((o >> 1) & 1);
          C.iz = 2 * t.boxes[b].iz + ((o >> 2) & 1);
          double w = t.root_width / std::ldexp(1.0, l + 1);
          C.center = corner + Vec3((C.ix + 0.5) * w, (C.iy + 0.5) * w, (C.iz + 0.5) * w);
          C.parent = b;
          for (auto& c : C.child) c = -1;
          C.begin = s; C.end = e; C.leaf = true; C.octant = o;
          t.boxes.push_back(C);
          t.boxes[b].child[o] = (int64_t)t.boxes.size() - 1;
          t.boxes[b].leaf = false;
        }
        s = e;
      }
    }
    int64_t next_end = (int64_t)t.boxes.size();
    if (next_end == next_begin) break;
    lvl_begin = next_begin; lvl_end = next_end;
  }
  t.leaves.clear();
  for (int64_t b = 0; b < (int64_t)t.boxes.size(); ++b)
    if (t.boxes[b].leaf) t.leaves.push_back(b);
  std::sort(t.leaves.begin(), t.leaves.end(),
            [&](int64_t a, int64_t b) { return t.boxes[a].begin < t.boxes[b].begin; });
}

// ---------------------------------------------------------------- wedges
int wedge_of(int64_t dx, int64_t dy, int64_t dz, int nf) {
  int64_t d[3] = {dx, dy, dz};
  int axis = 0;
  for (int a = 1; a < 3; ++a)
    if (std::llabs(d[a]) > std::llabs(d[axis])) axis = a;
  int face = 2 * axis + (d[axis] < 0 ? 1 : 0);
  int64_t da = std::llabs(d[axis]);
  int cells[2];
  int ci = 0;
  for (int a = 0; a < 3; ++a) {
    if (a == axis) continue;
    int64_t num = (d[a] + da) * nf, den = 2 * da;
    int64_t c = (num + den - 1) / den - 1;  // ceil(num/den) - 1: boundary → lower cell
    if (c < 0) c = 0;
    if (c > nf - 1) c = nf - 1;
    cells[ci++] = (int)c;
  }
  return face * nf * nf + cells[0] * nf + cells[1];
}

int anti_dir(int dir, int nf) {
  int face = dir / (nf * nf), rem = dir % (nf * nf);
  int c1 = rem / nf, c2 = rem % nf;
  return (face ^ 1) * nf * nf + (nf - 1 - c1) * nf + (nf - 1 - c2);
}

int child_dir(int dir, int nf) {
  int face = dir / (nf * nf), rem = dir % (nf * nf);
  int c1 = rem / nf, c2 = rem % nf;
  int h = nf / 2;
  return face * h * h + (c1 >> 1) * h + (c2 >> 1);
}

Vec3 dir_center(int dir, int nf) {
  int face = dir / (nf * nf), rem = dir % (nf * nf);
  int c1 = rem / nf, c2 = rem % nf;
  int axis = face / 2;
  double sgn = (face & 1) ? -1.0 : 1.0;
  double v[3];
  v[axis] = sgn;
  int ci = 0;
  for (int a = 0; a < 3; ++a) {
    if (a == axis) continue;
    int c = ci == 0 ? c1 : c2;
    v[a] = -1.0 + (2.0 * c + 1.0) / nf;
    ++ci;
  }
  Vec3 u(v[0], v[1], v[2]);
  return u * (1.0 / u.norm());
}

Mat3 rotation_to_z(const Vec3& u) {
  Mat3 R{};
  const Vec3 z(0, 0, 1);
  Vec3 ax = u.cross(z);
  double s = ax.norm(), c = u.dot(z);
  if (s < 1e-14) {
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) R.m[i][j] = (i == j) ? 1.0 : 0.0;
    if (c < 0) { R.m[1][1] = -1.0; R.m[2][2] = -1.0; }  // π about x
    return R;
  }
  Vec3 kx = ax * (1.0 / s);
  double K[3][3] = {{0, -kx.z, kx.y}, {kx.z, 0, -kx.x}, {-kx.y, kx.x, 0}};
  double kv[3] = {kx.x, kx.y, kx.z};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      R.m[i][j] = (i == j ? c : 0.0) + s * K[i][j] + (1.0 - c) * kv[i] * kv[j];
  return R;
}

}  // namespace fda
