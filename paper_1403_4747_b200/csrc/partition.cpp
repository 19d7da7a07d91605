// Sharding of the FDA over nranks GPUs.
//
// Leaves (Morton / tree order) are split into contiguous ranges balanced by
// an estimate of their downward + near-field work.  A rank keeps
//  * the S2M of its own leaves and the M2M ops whose child box intersects its
//    element range: its upward pass produces PARTIAL outgoing states (the
//    contribution of its own elements; the full state is the sum over the
//    ranks by linearity of S2M / M2M, Algorithm Step 2),
//  * the M2L (dense and §4.2 factored) and L2L ops whose destination is an
//    incoming state of a box that contains at least one of its leaves
//    (ancestors shared by several ranks are computed by each of them),
//  * the near field and L2T of its own leaves.
// Between the passes the ranks exchange partial outgoing states: rank r
// receives, from every other rank q contributing to an outgoing state that
// one of r's M2L ops reads, q's partial of that state (xrecv[q] / xsend[r],
// both sorted by state id, derived from the same global plan on every rank)
// and adds it to its own partial.  Its y rows are then exact for its elements
// and zero elsewhere; one all-reduce over the ranks forms the full y.  Every
// (target, source) pair of the operator is computed by exactly the rank that
// owns the target.
#include <algorithm>

#include "fda_internal.h"

namespace fda {

void apply_partition(const Params& p, const Tree& t, Plan& plan) {
  const int R = std::max(1, p.opt.nranks), r = p.opt.rank;
  const int64_t nleaf = (int64_t)plan.leaf_box.size();
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
  auto add_m2l = [&](int64_t dst_state, double flops) {
    const int64_t b = plan.in_states[dst_state].box;
    const int64_t li = leaf_of_box[b];
    if (li >= 0) w[li] += flops / 60.0;  // FP32 flops → near-evaluation equivalents
  };
  for (size_t l = 0; l < plan.m2l.size(); ++l)
    for (const Op& o : plan.m2l[l]) add_m2l(o.dst, 8.0 * plan.mats[o.mat].rows * plan.mats[o.mat].cols);
  for (const LrOp& o : plan.m2l_lr)
    add_m2l(o.dst, 16.0 * plan.mats[o.matV].rows * plan.mats[o.matV].cols);
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
  // ranks whose element range intersects [b, e): a contiguous run [lo, hi]
  auto ranks_of = [&](int64_t b, int64_t e, int& lo, int& hi) {
    lo = R; hi = -1;
    for (int k = 0; k < R; ++k)
      if (re0[k] < re1[k] && re0[k] < e && re1[k] > b) { lo = std::min(lo, k); hi = std::max(hi, k); }
  };
  const int64_t e0 = plan.own_e0, e1 = plan.own_e1;
  auto needed = [&](int64_t in_state) {
    const Box& B = t.boxes[plan.in_states[in_state].box];
    return B.begin < e1 && B.end > e0;
  };
  auto mine_out = [&](int64_t out_state) {
    const Box& B = t.boxes[plan.out_states[out_state].box];
    return B.begin < e1 && B.end > e0;
  };
  // exchange plan: for every M2L op, the ranks needing its destination (box ∩ range)
  // need the full source state, i.e. the partials of every contributing rank
  const int64_t nout = (int64_t)plan.out_states.size();
  std::vector<std::vector<int64_t>> need_by(R);   // out-states each rank reads in M2L
  {
    std::vector<std::vector<char>> mark(R, std::vector<char>(nout, 0));
    auto visit = [&](int64_t src, int64_t dst) {
      const Box& D = t.boxes[plan.in_states[dst].box];
      int lo, hi;
      ranks_of(D.begin, D.end, lo, hi);
      for (int k = lo; k <= hi; ++k) mark[k][src] = 1;
    };
    for (auto& lev : plan.m2l)
      for (const Op& o : lev) visit(o.src, o.dst);
    for (const LrOp& o : plan.m2l_lr) visit(o.src, o.dst);
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
      for (int q = lo; q <= hi; ++q) {
        if (q == k) continue;
        if (q == r) plan.xsend[k].push_back(sidx);   // I contribute a partial that k needs
        if (k == r) plan.xrecv[q].push_back(sidx);   // I need q's partial
      }
    }
  // partial upward pass: S2M of own leaves, M2M ops whose child box holds own elements
  for (int64_t i = 0; i < nleaf; ++i)
    if (i < plan.own_leaf0 || i >= plan.own_leaf1) {
      plan.leaf_S[i] = -1;
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
  for (auto& lev : plan.m2m) {
    std::vector<Op> keep;
    for (const Op& o : lev) if (mine_out(o.src)) keep.push_back(o);
    lev.swap(keep);
  }
  // L2T only for owned leaves
  for (int64_t i = 0; i < nleaf; ++i)
    if (i < plan.own_leaf0 || i >= plan.own_leaf1) plan.leaf_T[i] = -1;
}

}  // namespace fda
