#!/usr/bin/env python
"""W/X-list analysis of the direct (near-field) pairs of an adaptive tree.

    python tools/wx_lists.py [--config 4]

The FDA's Step 4 sends every leaf pair that no M2L covers to the
direct sum.  On a graded mesh (config 4: leaves on several levels) part of
those pairs are CROSS-LEVEL and NOT ADJACENT — the pairs KIFMM's W list
(source leaf finer than the target leaf: M2T) and X list (source leaf
coarser: S2L) would translate instead.  This tool counts, from the library's
own build tables, the direct element pairs by class and prices the two
options with the kernel costs measured here:
  direct: 3 Q3 evaluations per element pair (the near kernel's rate);
  M2T / S2L on the fly: one kernel evaluation per (element, equivalent point)
  of the far box (p_eq³ − (p_eq−2)³ = 296 points), i.e. n_B·296 (M2T) or
  n_C·296·3 (S2L) evaluations per pair — the same evaluation rate.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fda_inputs import config_mesh, CONFIGS  # noqa: E402
from paper_1403_4747_b200 import FDA  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    args = ap.parse_args()
    c = CONFIGS[args.config]
    V, F = config_mesh(args.config)
    f = FDA(V, F, c.k, c.alpha, c.eps)
    boxes = f.table("boxes").reshape(-1, 8)      # level, ix, iy, iz, parent, begin, end, leaf
    lr = f.table("leaf_range").reshape(-1, 2)
    nptr, nidx = f.table("near_ptr"), f.table("near_idx")
    leafb = np.nonzero(boxes[:, 7] == 1)[0]
    by_begin = {int(boxes[b, 5]): int(b) for b in leafb}
    lbox = np.array([by_begin[int(b)] for b in lr[:, 0]])
    lev = boxes[lbox, 0]
    ijk = boxes[lbox, 1:4]
    ne = lr[:, 1] - lr[:, 0]
    src = np.repeat(np.arange(len(lr)), np.diff(nptr))       # target leaf of each list entry
    dst = nidx
    lt, ls = lev[src], lev[dst]
    pairs = ne[src].astype(np.float64) * ne[dst]
    # adjacency at the finer level: the coarser box covers [2^d·i, 2^d·(i+1)) cells
    lf = np.maximum(lt, ls)
    dt, ds = lf - lt, lf - ls
    lo_t, hi_t = ijk[src] << dt[:, None], ((ijk[src] + 1) << dt[:, None]) - 1
    lo_s, hi_s = ijk[dst] << ds[:, None], ((ijk[dst] + 1) << ds[:, None]) - 1
    gap = np.maximum(lo_s - hi_t, lo_t - hi_s).max(axis=1)   # > 1: separated by at least one fine cell
    same = lt == ls
    cross_adj = (~same) & (gap <= 1)
    w_list = (~same) & (gap > 1) & (ls > lt)                  # source finer than target: M2T
    x_list = (~same) & (gap > 1) & (ls < lt)                  # source coarser: S2L
    p_eq = 8
    neq = p_eq ** 3 - (p_eq - 2) ** 3
    tot = pairs.sum()
    evals_direct = 3 * pairs
    ev_w = (ne[src] * neq)[w_list].sum()
    ev_x = (ne[dst] * 3 * neq)[x_list].sum()
    out = {"config": args.config, "N": len(F), "leaves": int(len(lr)), "leaf_levels": sorted(set(lev.tolist())),
           "direct_element_pairs": float(tot),
           "same_level": float(pairs[same].sum() / tot),
           "cross_level_adjacent": float(pairs[cross_adj].sum() / tot),
           "W_candidates (source finer, separated)": float(pairs[w_list].sum() / tot),
           "X_candidates (source coarser, separated)": float(pairs[x_list].sum() / tot),
           "direct_evals_of_W_X_pairs": float(evals_direct[w_list | x_list].sum()),
           "on_the_fly_M2T_S2L_evals": float(ev_w + ev_x),
           "verdict": None}
    d, m = out["direct_evals_of_W_X_pairs"], out["on_the_fly_M2T_S2L_evals"]
    out["saving_of_total_near_work"] = float((d - m) / evals_direct.sum()) if d > 0 else 0.0
    out["verdict"] = ("M2T/S2L would cut the near field by %.1f%%" % (100 * out["saving_of_total_near_work"])
                      if d > m else "direct is cheaper than on-the-fly M2T/S2L for these pairs")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
