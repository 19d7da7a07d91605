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
#include <map>
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

static inline int64_t skey(int64_t box, int dir) { return box * 65536 + (dir + 1); }

struct MatRegistry {
  std::map<std::vector<int64_t>, int64_t> ids;
  Plan* plan;
  int64_t get(const std::vector<int64_t>& key, const MatSpec& spec) {
    auto it = ids.find(key);
    if (it != ids.end()) return it->second;
    int64_t id = (int64_t)plan->specs.size();
    plan->specs.push_back(spec);
    ids.emplace(key, id);
    return id;
  }
};

void build_lists(const Geometry& g, const Params& p, Tree& t, Plan& plan) {
  (void)g;
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
      plan.near_idx.insert(plan.near_idx.end(), list.begin(), list.end());
      plan.near_ptr[i + 1] = (int64_t)plan.near_idx.size();
    }
  }

  // ---- M2L pairs and needed states
  std::vector<std::vector<std::pair<int64_t, int>>> out_need(nlev), in_need(nlev);
  struct RawPair { int64_t C, B; int u, w; };
  std::vector<std::vector<RawPair>> raw(nlev);
  for (int l = 1; l < nlev; ++l) {
    const Level& L = t.levels[l];
    for (int64_t b = L.box_begin; b < L.box_end; ++b) {
      const Box& B = t.boxes[b];
      for (int64_t c : IL[b]) {
        const Box& C = t.boxes[c];
        int u = -1, w = -1;
        if (L.hf) {
          u = wedge_of(B.ix - C.ix, B.iy - C.iy, B.iz - C.iz, L.nf);
          w = anti_dir(u, L.nf);
        }
        raw[l].push_back({c, b, u, w});
        out_need[l].push_back({c, u});
        in_need[l].push_back({b, w});
      }
    }
  }
  auto uniq = [](std::vector<std::pair<int64_t, int>>& v) {
    std::sort(v.begin(), v.end());
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

  // ---- state numbering
  plan.out_states.clear(); plan.in_states.clear();
  plan.out_level_begin.assign(nlev + 1, 0);
  plan.in_level_begin.assign(nlev + 1, 0);
  std::unordered_map<int64_t, int64_t> out_id, in_id;
  for (int l = 0; l < nlev; ++l) {
    plan.out_level_begin[l] = (int64_t)plan.out_states.size();
    for (auto& s : out_need[l]) {
      out_id[skey(s.first, s.second)] = (int64_t)plan.out_states.size();
      plan.out_states.push_back({s.first, s.second});
    }
    plan.in_level_begin[l] = (int64_t)plan.in_states.size();
    for (auto& s : in_need[l]) {
      in_id[skey(s.first, s.second)] = (int64_t)plan.in_states.size();
      plan.in_states.push_back({s.first, s.second});
    }
  }
  plan.out_level_begin[nlev] = (int64_t)plan.out_states.size();
  plan.in_level_begin[nlev] = (int64_t)plan.in_states.size();

  // ---- M2L ops
  for (int l = 0; l < nlev; ++l) {
    const Level& L = t.levels[l];
    for (auto& rp : raw[l]) {
      const Box& B = t.boxes[rp.B];
      const Box& C = t.boxes[rp.C];
      int64_t dx = B.ix - C.ix, dy = B.iy - C.iy, dz = B.iz - C.iz;
      std::vector<int64_t> key;
      if (L.hf) {
        // K depends only on t = R_u (c_D - c_C) (rotational invariance)
        Mat3 R = rotation_to_z(dir_center(rp.u, L.nf));
        Vec3 tv = R.apply(Vec3((double)dx, (double)dy, (double)dz));
        const double q = 1073741824.0;
        key = {MK_M2L, l, 1, std::llround(tv.x * q), std::llround(tv.y * q), std::llround(tv.z * q)};
      } else {
        key = {MK_M2L, l, 0, dx, dy, dz};
      }
      MatSpec sp{MK_M2L, l, 0, rp.u, -1, dx, dy, dz};
      int64_t m = reg.get(key, sp);
      plan.m2l[l].push_back({out_id.at(skey(rp.C, rp.u)), in_id.at(skey(rp.B, rp.w)), m});
    }
  }
  // ---- M2M (dst = parent out-state at level l) and L2L (src = parent in-state at level l)
  for (int l = 0; l + 1 < nlev; ++l) {
    const Level& L = t.levels[l];
    const Level& Lc = t.levels[l + 1];
    for (int64_t s = plan.out_level_begin[l]; s < plan.out_level_begin[l + 1]; ++s) {
      const State st = plan.out_states[s];
      const Box& P = t.boxes[st.box];
      if (P.leaf) continue;
      for (int o = 0; o < 8; ++o) {
        int64_t c = P.child[o];
        if (c < 0) continue;
        int d = Lc.hf ? child_dir(st.dir, L.nf) : -1;
        MatSpec sp{MK_M2M, l, o, st.dir, -1, 0, 0, 0};
        int64_t m = reg.get({MK_M2M, l, o, st.dir}, sp);
        plan.m2m[l].push_back({out_id.at(skey(c, d)), s, m});
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
        MatSpec sp{MK_L2L, l, o, st.dir, -1, 0, 0, 0};
        int64_t m = reg.get({MK_L2L, l, o, st.dir}, sp);
        plan.l2l[l].push_back({s, in_id.at(skey(c, d)), m});
      }
    }
  }
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
        const int64_t s = out_id.at(skey(b, u));
        plan.hf_s2m.push_back({i, s, reg.get({MK_S2M, b, u}, MatSpec{MK_S2M, l, 0, u, b, 0, 0, 0})});
        if (p.opt.rhs_operator)
          plan.hf_s2m_rhs.push_back(
              {i, s, reg.get({MK_S2M_RHS, b, u}, MatSpec{MK_S2M_RHS, l, 0, u, b, 0, 0, 0})});
      }
      auto li = std::lower_bound(in_need[l].begin(), in_need[l].end(), std::make_pair(b, -1));
      for (auto it = li; it != in_need[l].end() && it->first == b; ++it) {
        const int w = it->second;
        plan.hf_l2t.push_back({i, in_id.at(skey(b, w)), reg.get({MK_L2T, b, w}, MatSpec{MK_L2T, l, 0, w, b, 0, 0, 0})});
      }
      continue;
    }
    auto io = out_id.find(skey(b, -1));
    if (io != out_id.end()) {
      plan.leaf_out[i] = io->second;
      plan.leaf_S[i] = reg.get({MK_S2M, b}, MatSpec{MK_S2M, l, 0, -1, b, 0, 0, 0});
      if (p.opt.rhs_operator)
        plan.leaf_S_rhs[i] = reg.get({MK_S2M_RHS, b}, MatSpec{MK_S2M_RHS, l, 0, -1, b, 0, 0, 0});
    }
    auto ii = in_id.find(skey(b, -1));
    if (ii != in_id.end()) {
      plan.leaf_in[i] = ii->second;
      plan.leaf_T[i] = reg.get({MK_L2T, b}, MatSpec{MK_L2T, l, 0, -1, b, 0, 0, 0});
    }
  }
}

}  // namespace fda
