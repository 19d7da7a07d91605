#!/usr/bin/env python
"""Structure of the translation stages (M2M, L2L, M2L) of one config, for the
choice between op-stationary (one task per shared matrix, atomics into the
destinations) and destination-stationary formulations (one task per tile of
destination states accumulating every op into them, plain stores).

    python tools/xlate_structure.py --config 4 [--device 0] [--tile 128]

For each stage and level: ops, distinct matrices, destinations, sources,
ops per destination, ops per matrix; and, for a destination-stationary task
of `tile` consecutive destinations (tree order) that loops over the distinct
matrices its ops use, the FILL = ops / (tile × distinct matrices per tile) —
the fraction of the MMA columns that carry a real op (the rest are zero).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fda_inputs import config_mesh, CONFIGS  # noqa: E402
from paper_1403_4747_b200 import FDA  # noqa: E402


def fill(dst, key, tile, group=None):
    """ops / Σ_tiles (tile·#distinct keys in the tile); tiles of `tile` consecutive distinct dsts
    within a group (e.g. the wedge direction of the matrices: one tile never mixes groups)."""
    if group is None:
        group = np.zeros_like(dst)
    gd = np.unique(np.stack([group, dst]), axis=1)          # sorted (group, dst)
    gstart = np.r_[0, np.nonzero(np.diff(gd[0]))[0] + 1]
    pos = np.arange(gd.shape[1]) - np.repeat(gstart, np.diff(np.r_[gstart, gd.shape[1]]))
    tid_sorted = np.cumsum(np.r_[1, ((pos[1:] % tile) == 0) | (gd[0, 1:] != gd[0, :-1])]) - 1
    m = int(dst.max()) + 1
    t = tid_sorted[np.searchsorted(gd[0] * m + gd[1], group * m + dst)]
    pairs = np.unique(np.stack([t, key]), axis=1)
    return len(dst) / (pairs.shape[1] * tile), pairs.shape[1] / (t.max() + 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--tile", type=int, default=128)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    c = CONFIGS[args.config]
    V, F = config_mesh(args.config)
    t0 = time.time()
    f = FDA(V, F, c.k, c.alpha, c.eps, device=args.device)
    res = {"config": args.config, "build_s": round(time.time() - t0, 1), "tile": args.tile, "stages": []}
    mats = f.table("mats").reshape(-1, 3)
    specs = f.table("specs").reshape(-1, 8)
    for nm in ("m2m", "l2l", "m2l"):
        ops = f.table(nm).reshape(-1, 4)   # level, src, dst, mat
        for L in np.unique(ops[:, 0]):
            o = ops[ops[:, 0] == L]
            o = o[np.argsort(o[:, 2], kind="stable")]
            ud, cnt = np.unique(o[:, 2], return_counts=True)
            R, C = int(mats[o[0, 3], 1]), int(mats[o[0, 3], 2])
            # destination-stationary key: the matrix itself (a dst tile loops over its distinct matrices)
            fl, kpt = fill(o[:, 2], o[:, 3], args.tile, specs[o[:, 3], 3])
            d = dict(stage=nm, level=int(L), ops=len(o), mats=len(np.unique(o[:, 3])), dsts=len(ud),
                     srcs=len(np.unique(o[:, 1])), ops_per_dst=round(float(cnt.mean()), 2), max_ops_per_dst=int(cnt.max()),
                     R=R, C=C, gflop=round(8 * R * C * len(o) / 1e9, 3), ds_fill=round(fl, 3),
                     ds_mats_per_tile=round(float(kpt), 1))
            res["stages"].append(d)
            print(d, flush=True)
    lr = f.table("m2l_lr").reshape(-1, 6)   # level, src, dst, matV, matU, tmp
    for L in np.unique(lr[:, 0]):
        o = lr[lr[:, 0] == L]
        o = o[np.argsort(o[:, 2], kind="stable")]
        ud, cnt = np.unique(o[:, 2], return_counts=True)
        T, r = int(mats[o[0, 4], 1]), int(mats[o[0, 4], 2])
        g = specs[o[:, 4], 3]
        fl, kpt = fill(o[:, 2], o[:, 4], args.tile, g)
        fl64, _ = fill(o[:, 2], o[:, 4], 64, g)
        fl32, _ = fill(o[:, 2], o[:, 4], 32, g)
        rs = mats[o[:, 4], 2]
        d = dict(stage="m2l_lr", level=int(L), ops=len(o), mats=len(np.unique(o[:, 4])), dsts=len(ud),
                 srcs=len(np.unique(o[:, 1])), ops_per_dst=round(float(cnt.mean()), 1), T=T, r_mean=round(float(rs.mean()), 1),
                 gflop=round(float(16 * T * rs.sum()) / 1e9, 3), ds_fill=round(fl, 3), ds_fill64=round(fl64, 3),
                 ds_fill32=round(fl32, 3), ds_mats_per_tile=round(float(kpt), 1))
        res["stages"].append(d)
        print(d, flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh)


if __name__ == "__main__":
    main()
