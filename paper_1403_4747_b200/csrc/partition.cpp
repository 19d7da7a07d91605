// Sharding of the FDA over nranks GPUs (SURVEY §8(e), round-1 design).
//
// Leaves (Morton / tree order) are split into contiguous ranges balanced by
// an estimate of their downward + near-field work.  A rank keeps
//  * every S2M and M2M op (the upward pass is replicated: it is ~15% of the
//    matvec and needs no exchange of outgoing states),
//  * the M2L (dense and §4.2 factored) and L2L ops whose destination is an
//    incoming state of a box that contains at least one of its leaves
//    (ancestors shared by several ranks are computed by each of them),
//  * the near field and L2T of its own leaves.
// Its y rows are therefore exact for its elements and zero elsewhere; one
// all-reduce over the ranks forms the full y.  Every (target, source) pair of
// the operator is computed by exactly the rank that owns the target.
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
  const int64_t e0 = plan.own_e0, e1 = plan.own_e1;
  auto needed = [&](int64_t in_state) {
    const Box& B = t.boxes[plan.in_states[in_state].box];
    return B.begin < e1 && B.end > e0;
  };
  for (auto& lev : plan.m2l) {
    std::vector<Op> keep;
    for (const Op& o : lev) if (needed(o.dst)) keep.push_back(o);
    lev.swap(keep);
  }
  {
    std::vector<LrOp> keep;
    for (const LrOp& o : plan.m2l_lr) if (needed(o.dst)) keep.push_back(o);
    plan.m2l_lr.swap(keep);
  }
  for (auto& lev : plan.l2l) {
    std::vector<Op> keep;
    for (const Op& o : lev) if (needed(o.dst)) keep.push_back(o);
    lev.swap(keep);
  }
  // L2T only for owned leaves
  for (int64_t i = 0; i < nleaf; ++i)
    if (i < plan.own_leaf0 || i >= plan.own_leaf1) plan.leaf_T[i] = -1;
}

}  // namespace fda
