// Sharding of the FDA over nranks GPUs.
//
// Runs right after the lists (before any operator table is built), so that a
// rank builds, uploads and applies only its share.  Leaves (Morton / tree
// order) are split into contiguous ranges balanced by an estimate of their
// near-field and downward work.  A rank keeps
//  * the S2M of its own leaves and the M2M ops whose child box intersects its
//    element range: its upward pass produces PARTIAL outgoing states (the
//    contribution of its own elements; the full state is the sum over the
//    ranks by linearity of S2M / M2M, Algorithm Step 2),
//  * the M2L ops whose destination is an incoming state of a box that contains
//    at least one of its elements, and the L2L ops into such boxes (ancestors
//    shared by several ranks are computed by each of them),
//  * the near field, the correction rows and the L2T of its own leaves,
//  * only the matrices those ops read (needed[id]).
// Between the passes the ranks exchange partial outgoing states: rank r
// receives, from every other rank q contributing to an outgoing state that
// one of r's M2L ops reads, q's partial of that state (xrecv[q] / xsend[r],
// both sorted by state id, derived from the same GLOBAL op list on every
// rank before pruning) and adds it to its own partial.  Its y rows are then
// exact for its elements and zero elsewhere.  Every (target, source) pair of
// the operator is computed by exactly the rank that owns the target.
#include <algorithm>

#include "fda_internal.h"

namespace fda {

void apply_partition(const Params& p, const Tree& t, Plan& plan, std::vector<char>& needed) {
  const int R = std::max(1, p.opt.nranks), r = p.opt.rank;
  const int64_t nleaf = (int64_t)plan.leaf_box.size();
  needed.assign(plan.specs.size(), 1);
  // per level: M2L ops per distinct K̃ over the whole tree (the §4.2 routing rule, fda_api.cpp)
  plan.m2l_share.assign(plan.m2l.size(), 0.0);
  for (size_t l = 0; l < plan.m2l.size(); ++l) {
    std::vector<int64_t> mats;
    mats.reserve(plan.m2l[l].size());
    for (const Op& o : plan.m2l[l]) mats.push_back(o.mat);
    std::sort(mats.begin(), mats.end());
    const int64_t nd = (int64_t)(std::unique(mats.begin(), mats.end()) - mats.begin());
    plan.m2l_share[l] = nd ? (double)plan.m2l[l].size() / (double)nd : 0.0;
  }
  if (R <= 1) {
    plan.own_leaf0 = 0; plan.own_leaf1 = nleaf;
    plan.own_e0 = 0; plan.own_e1 = nleaf ? t.boxes[plan.leaf_box[nleaf - 1]].end : 0;
    return;
  }
  // per-leaf work: near-field evaluations + corrections + leaf-level M2L (as evaluation equivalents)
  std::vector<double> w(nleaf, 0.0);
  std::vector<int64_t> leaf_of_box(t.boxes.size(), -1);
  for (int64_t i = 0; i < nleaf; ++i) leaf_of_box[plan.leaf_box[i]] = i;
  for (int64_t i = 0; i < nleaf; ++i) {
    const Box& B = t.boxes[plan.leaf_box[i]];
    int64_t srcs = 0;
    for (int64_t e = plan.near_ptr[i]; e < plan.near_ptr[i + 1]; ++e) {
      const Box& C = t.boxes[plan.leaf_box[plan.near_idx[e]]];
      srcs += C.end - C.begin;
    }
    w[i] = 3.0 * (double)(B.end - B.begin) * (double)srcs + (double)(B.end - B.begin) * 80.0;
  }
  // M2L work of every box, attributed to the leaves below it in proportion to their elements
  // (8·T² flops per op; the §4.2 factorisation is decided later and scales every level alike)
  {
    std::vector<double> box_fl(t.boxes.size(), 0.0);
    for (size_t l = 0; l < plan.m2l.size(); ++l) {
      const double T = t.levels[l].rank;
      for (const Op& o : plan.m2l[l]) box_fl[plan.in_states[o.dst].box] += 8.0 * T * T;
    }
    for (int64_t i = 0; i < nleaf; ++i) {
      const int64_t b = plan.leaf_box[i];
      const double ne = (double)(t.boxes[b].end - t.boxes[b].begin);
      for (int64_t a = b; a >= 0; a = t.boxes[a].parent) {
        const double na = (double)(t.boxes[a].end - t.boxes[a].begin);
        if (box_fl[a] > 0) w[i] += box_fl[a] * ne / na / 60.0;   // FP32 flops → near-evaluation equivalents
      }
    }
  }
  double total = 0;
  for (double v : w) total += v;
  // contiguous split: rank q starts at the first leaf whose prefix work exceeds q·total/R
  std::vector<int64_t> start(R + 1, nleaf);
  start[0] = 0;
  double acc = 0;
  int q = 1;
  for (int64_t i = 0; i < nleaf && q < R; ++i) {
    acc += w[i];
    while (q < R && acc >= total * q / R) start[q++] = i + 1;
  }
  for (int k = 1; k <= R; ++k) start[k] = std::max(start[k], start[k - 1]);
  plan.own_leaf0 = start[r];
  plan.own_leaf1 = start[r + 1];
  plan.own_e0 = plan.own_leaf0 < nleaf ? t.boxes[plan.leaf_box[plan.own_leaf0]].begin : 0;
  plan.own_e1 = plan.own_leaf1 > plan.own_leaf0 ? t.boxes[plan.leaf_box[plan.own_leaf1 - 1]].end : plan.own_e0;
  // element range of every rank (contiguous, in rank order; empty ranks have e0 = e1)
  std::vector<int64_t> re0(R), re1(R);
  for (int k = 0; k < R; ++k) {
    re0[k] = start[k] < nleaf ? t.boxes[plan.leaf_box[start[k]]].begin : (nleaf ? t.boxes[plan.leaf_box[nleaf - 1]].end : 0);
    re1[k] = start[k + 1] > start[k] ? t.boxes[plan.leaf_box[start[k + 1] - 1]].end : re0[k];
  }
  plan.rank_e0 = re0;
  plan.rank_e1 = re1;
  // ranks whose element range intersects [b, e): a contiguous run [lo, hi]
  auto ranks_of = [&](int64_t b, int64_t e, int& lo, int& hi) {
    lo = R; hi = -1;
    for (int k = 0; k < R; ++k)
      if (re0[k] < re1[k] && re0[k] < e && re1[k] > b) { lo = std::min(lo, k); hi = std::max(hi, k); }
  };
  const int64_t e0 = plan.own_e0, e1 = plan.own_e1;
  auto mine_in = [&](int64_t in_state) {
    const Box& B = t.boxes[plan.in_states[in_state].box];
    return B.begin < e1 && B.end > e0;
  };
  auto mine_out = [&](int64_t out_state) {
    const Box& B = t.boxes[plan.out_states[out_state].box];
    return B.begin < e1 && B.end > e0;
  };
  // exchange plan from the GLOBAL M2L op list (identical on every rank): for every op, the
  // ranks needing its destination (box ∩ range) need the full source state, i.e. the
  // partials of every contributing rank
  const int64_t nout = (int64_t)plan.out_states.size();
  std::vector<std::vector<int64_t>> need_by(R);   // out-states each rank reads in M2L
  {
    std::vector<std::vector<char>> mark(R, std::vector<char>(nout, 0));
    for (auto& lev : plan.m2l)
      for (const Op& o : lev) {
        const Box& D = t.boxes[plan.in_states[o.dst].box];
        int lo, hi;
        ranks_of(D.begin, D.end, lo, hi);
        for (int k = lo; k <= hi; ++k) mark[k][o.src] = 1;
      }
    for (int k = 0; k < R; ++k)
      for (int64_t sidx = 0; sidx < nout; ++sidx)
        if (mark[k][sidx]) need_by[k].push_back(sidx);
  }
  plan.xsend.assign(R, {});
  plan.xrecv.assign(R, {});
  for (int k = 0; k < R; ++k)
    for (int64_t sidx : need_by[k]) {
      const Box& B = t.boxes[plan.out_states[sidx].box];
      int lo, hi;
      ranks_of(B.begin, B.end, lo, hi);
      for (int qq = lo; qq <= hi; ++qq) {
        if (qq == k) continue;
        if (qq == r) plan.xsend[k].push_back(sidx);   // I contribute a partial that k needs
        if (k == r) plan.xrecv[qq].push_back(sidx);   // I need qq's partial
      }
    }
  // this rank's ops: partial upward pass (S2M of own leaves, M2M whose child box holds own
  // elements), downward pass into boxes holding own elements (M2L, L2L), L2T of own leaves
  for (int64_t i = 0; i < nleaf; ++i)
    if (i < plan.own_leaf0 || i >= plan.own_leaf1) {
      plan.leaf_S[i] = -1;
      plan.leaf_T[i] = -1;
      if (!plan.leaf_S_rhs.empty()) plan.leaf_S_rhs[i] = -1;
    }
  auto own_ops = [&](std::vector<LeafOp>& v) {
    std::vector<LeafOp> keep;
    for (const LeafOp& o : v)
      if (o.leaf >= plan.own_leaf0 && o.leaf < plan.own_leaf1) keep.push_back(o);
    v.swap(keep);
  };
  own_ops(plan.hf_s2m);
  own_ops(plan.hf_s2m_rhs);
  own_ops(plan.hf_l2t);
  auto prune = [&](std::vector<std::vector<Op>>& ops, bool by_src_out) {
    for (auto& lev : ops) {
      std::vector<Op> keep;
      for (const Op& o : lev)
        if (by_src_out ? mine_out(o.src) : mine_in(o.dst)) keep.push_back(o);
      lev.swap(keep);
    }
  };
  prune(plan.m2m, true);
  prune(plan.m2l, false);
  prune(plan.l2l, false);
  // the matrices these ops read
  needed.assign(plan.specs.size(), 0);
  for (auto* ops : {&plan.m2m, &plan.m2l, &plan.l2l})
    for (auto& lev : *ops)
      for (const Op& o : lev) needed[o.mat] = 1;
  for (int64_t i = 0; i < nleaf; ++i) {
    if (plan.leaf_S[i] >= 0) needed[plan.leaf_S[i]] = 1;
    if (plan.leaf_T[i] >= 0) needed[plan.leaf_T[i]] = 1;
    if (!plan.leaf_S_rhs.empty() && plan.leaf_S_rhs[i] >= 0) needed[plan.leaf_S_rhs[i]] = 1;
  }
  for (auto* v : {&plan.hf_s2m, &plan.hf_s2m_rhs, &plan.hf_l2t})
    for (const LeafOp& o : *v) needed[o.mat] = 1;
}

}  // namespace fda
