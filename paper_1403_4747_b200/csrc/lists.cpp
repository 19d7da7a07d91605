// Interaction lists, direct (near) lists, directional states and the
// translation op lists (host).  PAPER.md Algorithm Step 1.5 and the
// pass structure of Steps 2-4; readings C9-C11, C17, C18.
//
// N(B)  = {X at level l : ¬adm_l(B, X)}   (computed top-down: N(B) ⊆ children(N(parent)))
// IL(B) = {X ∈ children(N(parent(B))) : adm_l(B, X)}   — the M2L sources of B.
// adm is hereditary, so every ordered element pair is covered exactly once:
// by one M2L between ancestors, or by a direct leaf pair.
#include <algorithm>
#include <cmath>
#include <array>
#include <parallel/algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <stdexcept>
#include <tuple>
#include <unordered_map>

#include "fda_internal.h"

namespace fda {

static bool adm(const Tree& t, int l, const Box& a, const Box& b) {
  int64_t dx = a.ix - b.ix, dy = a.iy - b.iy, dz = a.iz - b.iz;
  int64_t cheb = std::max({std::llabs(dx), std::llabs(dy), std::llabs(dz)});
  if (cheb < 2) return false;
  const Level& L = t.levels[l];
  if (!L.hf) return true;
  // ‖Δc‖ ≥ w²/λ  ⇔  (dx²+dy²+dz²) ≥ (w/λ)²   (offsets in units of w)
  double r = L.width / t.lambda;
  return double(dx * dx + dy * dy + dz * dz) >= r * r;
}

// matrix identity key (kind, level / box, …): ≤ 6 integers, hashed
using MKey = std::array<int64_t, 6>;
struct MKeyHash {
  size_t operator()(const MKey& k) const {
    uint64_t h = 0x9e3779b97f4a7c15ull;
    for (int64_t v : k) h = (h ^ (uint64_t)v) * 0x100000001b3ull + (h >> 29);
    return (size_t)h;
  }
};
struct MatRegistry {
  std::unordered_map<MKey, int64_t, MKeyHash> ids;
  Plan* plan;
  int64_t get(std::initializer_list<int64_t> key, const MatSpec& spec) {
    MKey k{};
    k.fill(INT64_MIN);
    size_t i = 0;
    for (int64_t v : key) k[i++] = v;
    return get(k, spec);
  }
  int64_t get(const MKey& k, const MatSpec& spec) {
    auto it = ids.find(k);
    if (it != ids.end()) return it->second;
    int64_t id = (int64_t)plan->specs.size();
    plan->specs.push_back(spec);
    ids.emplace(k, id);
    return id;
  }
};


void build_lists(const Geometry& g, const Params& p, Tree& t, Plan& plan) {
  (void)g;
  auto tp = std::chrono::steady_clock::now();
  auto mark = [&](const char* name) {
    auto now = std::chrono::steady_clock::now();
    if (p.opt.verbose > 1) fprintf(stderr, "  [lists] %-10s %8.3f s\n", name, std::chrono::duration<double>(now - tp).count());
    tp = now;
  };
  const int nlev = (int)t.levels.size();
  const int64_t nb = (int64_t)t.boxes.size();
  plan.m2m.assign(nlev, {});
  plan.m2l.assign(nlev, {});
  plan.l2l.assign(nlev, {});
  plan.specs.clear();
  MatRegistry reg{{}, &plan};

  // ---- direct lists
  const int64_t nleaf = (int64_t)t.leaves.size();
  std::vector<int64_t> leaf_index(nb, -1);
  for (int64_t i = 0; i < nleaf; ++i) leaf_index[t.leaves[i]] = i;
  plan.leaf_box = t.leaves;
  plan.near_ptr.assign(nleaf + 1, 0);
  plan.near_idx.clear();

  if (p.opt.direct_all) {
    for (int64_t i = 0; i < nleaf; ++i) {
      for (int64_t j = 0; j < nleaf; ++j) plan.near_idx.push_back(j);
      plan.near_ptr[i + 1] = (int64_t)plan.near_idx.size();
    }
  }

  std::vector<std::vector<int64_t>> N(nb), IL(nb);
  if (!p.opt.direct_all) {
    N[0].push_back(0);
    for (int l = 1; l < nlev; ++l) {
      for (int64_t b = t.levels[l].box_begin; b < t.levels[l].box_end; ++b) {
        const Box& B = t.boxes[b];
        for (int64_t X : N[B.parent]) {
          for (int o = 0; o < 8; ++o) {
            int64_t c = t.boxes[X].child[o];
            if (c < 0) continue;
            if (adm(t, l, B, t.boxes[c])) IL[b].push_back(c);
            else N[b].push_back(c);
          }
        }
      }
    }
    std::vector<std::vector<int64_t>> lists(nleaf);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < nleaf; ++i) {
      const int64_t b = t.leaves[i];
      std::vector<int64_t> anc;
      for (int64_t a = b; a >= 0; a = t.boxes[a].parent) anc.push_back(a);
      std::reverse(anc.begin(), anc.end());  // anc[l] = ancestor at level l
      std::vector<int64_t> list;
      const int lb = t.boxes[b].level;
      for (int l = 0; l <= lb; ++l) {
        for (int64_t X : N[anc[l]]) {
          if (t.boxes[X].leaf) list.push_back(leaf_index[X]);
          else if (l == lb) {
            // all leaves below X are direct partners of B (coarser-B pairs)
            std::vector<int64_t> st{X};
            while (!st.empty()) {
              int64_t y = st.back(); st.pop_back();
              if (t.boxes[y].leaf) { list.push_back(leaf_index[y]); continue; }
              for (int o = 0; o < 8; ++o) if (t.boxes[y].child[o] >= 0) st.push_back(t.boxes[y].child[o]);
            }
          }
        }
      }
      std::sort(list.begin(), list.end());
      list.erase(std::unique(list.begin(), list.end()), list.end());
      lists[i].swap(list);
    }
    for (int64_t i = 0; i < nleaf; ++i) {
      plan.near_idx.insert(plan.near_idx.end(), lists[i].begin(), lists[i].end());
      plan.near_ptr[i + 1] = (int64_t)plan.near_idx.size();
      std::vector<int64_t>().swap(lists[i]);
    }
  }

  mark("direct");
  // ---- M2L pairs and needed states
  std::vector<std::vector<std::pair<int64_t, int>>> out_need(nlev), in_need(nlev);
  struct RawPair { int64_t C, B; int u, w; };
  std::vector<std::vector<RawPair>> raw(nlev);
  for (int l = 1; l < nlev; ++l) {
    const Level& L = t.levels[l];
    const int64_t nbl = L.box_end - L.box_begin;
    std::vector<int64_t> start(nbl + 1, 0);
    for (int64_t b = 0; b < nbl; ++b) start[b + 1] = start[b] + (int64_t)IL[L.box_begin + b].size();
    raw[l].resize(start[nbl]);
    out_need[l].resize(start[nbl]);
    in_need[l].resize(start[nbl]);
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t bi = 0; bi < nbl; ++bi) {
      const int64_t b = L.box_begin + bi;
      const Box& B = t.boxes[b];
      int64_t q = start[bi];
      for (int64_t c : IL[b]) {
        const Box& C = t.boxes[c];
        int u = -1, w = -1;
        if (L.hf) {
          u = wedge_of(B.ix - C.ix, B.iy - C.iy, B.iz - C.iz, L.nf);
          w = anti_dir(u, L.nf);
        }
        raw[l][q] = {c, b, u, w};
        out_need[l][q] = {c, u};
        in_need[l][q] = {b, w};
        ++q;
      }
    }
  }
  auto uniq = [](std::vector<std::pair<int64_t, int>>& v) {
    __gnu_parallel::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  };
  for (int l = 0; l < nlev; ++l) {
    uniq(out_need[l]);
    uniq(in_need[l]);
    if (l + 1 >= nlev) break;
    const Level& L = t.levels[l];
    const Level& Lc = t.levels[l + 1];
    for (auto* need : {&out_need, &in_need}) {
      for (auto& s : (*need)[l]) {
        const Box& P = t.boxes[s.first];
        if (P.leaf) continue;
        for (int o = 0; o < 8; ++o) {
          int64_t c = P.child[o];
          if (c < 0) continue;
          int d = Lc.hf ? child_dir(s.second, L.nf) : -1;
          (*need)[l + 1].push_back({c, d});
        }
      }
    }
  }

  mark("need");
  // ---- state numbering
  plan.out_states.clear(); plan.in_states.clear();
  plan.out_level_begin.assign(nlev + 1, 0);
  plan.in_level_begin.assign(nlev + 1, 0);
  for (int l = 0; l < nlev; ++l) {
    plan.out_level_begin[l] = (int64_t)plan.out_states.size();
    for (auto& s : out_need[l]) plan.out_states.push_back({s.first, s.second});
    plan.in_level_begin[l] = (int64_t)plan.in_states.size();
    for (auto& s : in_need[l]) plan.in_states.push_back({s.first, s.second});
  }
  // per level and box: first index of its states in the level's sorted need list (O(1) + a short
  // search over the box's directions instead of a search over the whole level)
  auto firsts = [&](const std::vector<std::vector<std::pair<int64_t, int>>>& need) {
    std::vector<std::vector<int64_t>> f(nlev);
    for (int l = 0; l < nlev; ++l) {
      const int64_t b0 = t.levels[l].box_begin, nbl = t.levels[l].box_end - b0;
      f[l].assign(nbl + 1, 0);
      for (const auto& s : need[l]) ++f[l][s.first - b0 + 1];
      for (int64_t b = 0; b < nbl; ++b) f[l][b + 1] += f[l][b];
    }
    return f;
  };
  const auto out_first = firsts(out_need), in_first = firsts(in_need);
  auto lookup = [&](const std::vector<std::pair<int64_t, int>>& need, const std::vector<int64_t>& first, int64_t begin,
                    int l, int64_t box, int dir) {
    const int64_t bi = box - t.levels[l].box_begin;
    auto lo = need.begin() + first[bi], hi = need.begin() + first[bi + 1];
    auto it = std::lower_bound(lo, hi, std::make_pair(box, dir));
    if (it == hi || it->second != dir) throw std::runtime_error("missing FDA state");
    return begin + (int64_t)(it - need.begin());
  };
  auto out_id = [&](int l, int64_t box, int dir) {
    return lookup(out_need[l], out_first[l], plan.out_level_begin[l], l, box, dir);
  };
  auto in_id = [&](int l, int64_t box, int dir) {
    return lookup(in_need[l], in_first[l], plan.in_level_begin[l], l, box, dir);
  };
  plan.out_level_begin[nlev] = (int64_t)plan.out_states.size();
  plan.in_level_begin[nlev] = (int64_t)plan.in_states.size();

  mark("states");
  // ---- M2L ops: keys and state ids in parallel, matrix ids assigned in pair order (serial)
  for (int l = 0; l < nlev; ++l) {
    const Level& L = t.levels[l];
    const int64_t np = (int64_t)raw[l].size();
    if (!np) continue;
    std::vector<Mat3> Rdir(L.hf ? L.ndir : 0);
    for (int u = 0; u < (int)Rdir.size(); ++u) Rdir[u] = rotation_to_z(dir_center(u, L.nf));
    std::vector<MKey> keys(np);
    plan.m2l[l].resize(np);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < np; ++i) {
      const RawPair& rp = raw[l][i];
      const Box& B = t.boxes[rp.B];
      const Box& C = t.boxes[rp.C];
      const int64_t dx = B.ix - C.ix, dy = B.iy - C.iy, dz = B.iz - C.iz;
      if (L.hf) {
        // K depends only on t = R_u (c_D - c_C) (rotational invariance)
        const Vec3 tv = Rdir[rp.u].apply(Vec3((double)dx, (double)dy, (double)dz));
        const double q = 1073741824.0;
        keys[i] = MKey{MK_M2L, l, 1, std::llround(tv.x * q), std::llround(tv.y * q), std::llround(tv.z * q)};
      } else {
        keys[i] = MKey{MK_M2L, l, 0, dx, dy, dz};
      }
      plan.m2l[l][i] = {out_id(l, rp.C, rp.u), in_id(l, rp.B, rp.w), -1};
    }
    // (u, offset) → matrix id cache (many pairs share a wedge and an offset); the full key
    // (rotated offset) only on a miss
    std::unordered_map<uint64_t, int64_t> fast;
    for (int64_t i = 0; i < np; ++i) {
      const RawPair& rp = raw[l][i];
      const Box& B = t.boxes[rp.B];
      const Box& C = t.boxes[rp.C];
      const int64_t dx = B.ix - C.ix, dy = B.iy - C.iy, dz = B.iz - C.iz;
      const uint64_t fk = ((uint64_t)(rp.u + 1) << 42) | ((uint64_t)(dx & 0x3fff) << 28) |
                          ((uint64_t)(dy & 0x3fff) << 14) | (uint64_t)(dz & 0x3fff);
      const bool inr = std::llabs(dx) < 8192 && std::llabs(dy) < 8192 && std::llabs(dz) < 8192;
      if (inr) {
        auto it = fast.find(fk);
        if (it != fast.end()) {
          plan.m2l[l][i].mat = it->second;
          continue;
        }
      }
      MatSpec sp{MK_M2L, l, 0, rp.u, -1, dx, dy, dz};
      plan.m2l[l][i].mat = reg.get(keys[i], sp);
      if (inr) fast[fk] = plan.m2l[l][i].mat;
    }
  }
  mark("m2l");
  // ---- M2M (dst = parent out-state at level l) and L2L (src = parent in-state at level l)
  for (int l = 0; l + 1 < nlev; ++l) {
    const Level& L = t.levels[l];
    const Level& Lc = t.levels[l + 1];
    // (kind, octant, dir) → matrix id at this level (registry lookups only on first use)
    std::vector<int64_t> cache(2 * 8 * (size_t)(L.ndir + 1), -1);
    auto mat_of = [&](int kind, int o, int dir) {
      int64_t& c = cache[((size_t)(kind == MK_M2M ? 0 : 1) * 8 + o) * (L.ndir + 1) + (dir + 1)];
      if (c < 0) c = reg.get({kind, l, o, dir}, MatSpec{kind, l, o, dir, -1, 0, 0, 0});
      return c;
    };
    for (int64_t s = plan.out_level_begin[l]; s < plan.out_level_begin[l + 1]; ++s) {
      const State st = plan.out_states[s];
      const Box& P = t.boxes[st.box];
      if (P.leaf) continue;
      for (int o = 0; o < 8; ++o) {
        int64_t c = P.child[o];
        if (c < 0) continue;
        int d = Lc.hf ? child_dir(st.dir, L.nf) : -1;
        plan.m2m[l].push_back({out_id(l + 1, c, d), s, mat_of(MK_M2M, o, st.dir)});
      }
    }
    for (int64_t s = plan.in_level_begin[l]; s < plan.in_level_begin[l + 1]; ++s) {
      const State st = plan.in_states[s];
      const Box& P = t.boxes[st.box];
      if (P.leaf) continue;
      for (int o = 0; o < 8; ++o) {
        int64_t c = P.child[o];
        if (c < 0) continue;
        int d = Lc.hf ? child_dir(st.dir, L.nf) : -1;
        plan.l2l[l].push_back({s, in_id(l + 1, c, d), mat_of(MK_L2L, o, st.dir)});
      }
    }
  }
  mark("m2m/l2l");
  // ---- leaves: S2M / L2T
  plan.leaf_S.assign(nleaf, -1); plan.leaf_T.assign(nleaf, -1); plan.leaf_S_rhs.assign(nleaf, -1);
  plan.leaf_out.assign(nleaf, -1); plan.leaf_in.assign(nleaf, -1);
  plan.hf_s2m.clear(); plan.hf_s2m_rhs.clear(); plan.hf_l2t.clear();
  for (int64_t i = 0; i < nleaf; ++i) {
    const int64_t b = t.leaves[i];
    const int l = t.boxes[b].level;
    if (t.levels[l].hf) {
      // HF leaf (opt.hf_leaves): directional S2M for every used outgoing wedge u and
      // L2T for every incoming wedge w (Algorithm Step 2/3 leaf branches)
      auto lo = std::lower_bound(out_need[l].begin(), out_need[l].end(), std::make_pair(b, -1));
      for (auto it = lo; it != out_need[l].end() && it->first == b; ++it) {
        const int u = it->second;
        const int64_t s = out_id(l, b, u);
        plan.hf_s2m.push_back({i, s, reg.get({MK_S2M, b, u}, MatSpec{MK_S2M, l, 0, u, b, 0, 0, 0})});
        if (p.opt.rhs_operator)
          plan.hf_s2m_rhs.push_back(
              {i, s, reg.get({MK_S2M_RHS, b, u}, MatSpec{MK_S2M_RHS, l, 0, u, b, 0, 0, 0})});
      }
      auto li = std::lower_bound(in_need[l].begin(), in_need[l].end(), std::make_pair(b, -1));
      for (auto it = li; it != in_need[l].end() && it->first == b; ++it) {
        const int w = it->second;
        plan.hf_l2t.push_back({i, in_id(l, b, w), reg.get({MK_L2T, b, w}, MatSpec{MK_L2T, l, 0, w, b, 0, 0, 0})});
      }
      continue;
    }
    auto has = [](const std::vector<std::pair<int64_t, int>>& need, int64_t box) {
      return std::binary_search(need.begin(), need.end(), std::make_pair(box, -1));
    };
    if (has(out_need[l], b)) {
      plan.leaf_out[i] = out_id(l, b, -1);
      plan.leaf_S[i] = reg.get({MK_S2M, b}, MatSpec{MK_S2M, l, 0, -1, b, 0, 0, 0});
      if (p.opt.rhs_operator)
        plan.leaf_S_rhs[i] = reg.get({MK_S2M_RHS, b}, MatSpec{MK_S2M_RHS, l, 0, -1, b, 0, 0, 0});
    }
    if (has(in_need[l], b)) {
      plan.leaf_in[i] = in_id(l, b, -1);
      plan.leaf_T[i] = reg.get({MK_L2T, b}, MatSpec{MK_L2T, l, 0, -1, b, 0, 0, 0});
    }
  }
}

}  // namespace fda
