"""Config 5 (BASELINE configs[4]): icosphere s=9, N = 5,242,880, kD = 1000,
ε = 1e-4 on one B200: build, matvec time, and parity on 2,000 seeded oracle
rows.  One JSON line.

    python tools/config5.py [--rows 2000] [--cfg 5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _level_stats(f):
    """Per level and translation stage: ops, distinct matrices, shape, GFLOP."""
    mats = f.table("mats").reshape(-1, 3)
    out = {}
    for stage in ("m2m", "m2l", "l2l"):
        ops = f.table(stage).reshape(-1, 4)
        for l in sorted(set(ops[:, 0].tolist())):
            o = ops[ops[:, 0] == l]
            rc = mats[o[:, 3], 1] * mats[o[:, 3], 2]
            out[f"{stage}_L{l}"] = {"ops": int(len(o)), "mats": int(len(set(o[:, 3].tolist()))),
                                    "rows": int(mats[o[0, 3], 1]), "cols": int(mats[o[0, 3], 2]),
                                    "gflop": round(8 * float(rc.sum()) / 1e9, 3)}
    lr = f.table("m2l_lr").reshape(-1, 6)
    for l in sorted(set(lr[:, 0].tolist())):
        o = lr[lr[:, 0] == l]
        r, T = mats[o[:, 3], 1], mats[o[:, 3], 2]
        out[f"m2l_lr_L{l}"] = {"ops": int(len(o)), "mats": int(len(set(o[:, 3].tolist()))), "T": int(T[0]),
                               "r_mean": round(float(r.mean()), 1), "r_max": int(r.max()),
                               "gflop": round(16 * float((r * T).sum()) / 1e9, 3)}
    return out


def main():
    import torch
    from fda_inputs import config_mesh, CONFIGS, random_density, sampled_rows
    from paper_1403_4747_b200 import FDA
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--rows", type=int, default=2000)
    ap.add_argument("--tc", type=int, default=2)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--solve", action="store_true", help="also bm_solve the plane-wave system (GMRES tol 1e-4)")
    ap.add_argument("--max-iter", type=int, default=400)
    ap.add_argument("--restart", type=int, default=0)
    ap.add_argument("--lrtc", type=int, default=2, help="opt.lr_tensor_cores (fused tcgen05 factored M2L; 2 = library default)")
    a = ap.parse_args()
    c = CONFIGS[a.cfg]
    t0 = time.perf_counter()
    V, F = config_mesh(a.cfg)
    t_mesh = time.perf_counter() - t0
    N = len(F)
    t0 = time.perf_counter()
    f = FDA(V, F, c.k, c.alpha, c.eps, verbose=1, tensor_cores=a.tc, lr_tensor_cores=a.lrtc)
    t_build = time.perf_counter() - t0
    st = f.stats()
    levels = _level_stats(f)
    x = random_density(N, c.x_seed)
    xd = torch.from_numpy(x.astype(np.complex64)).cuda()
    yd = torch.empty_like(xd)
    for _ in range(3):
        f.matvec(xd, yd)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        f.matvec(xd, yd)
    e.record()
    torch.cuda.synchronize()
    mv_ms = s.elapsed_time(e) / 10
    f.set_profiling(True)
    f.matvec(xd, yd)
    torch.cuda.synchronize()
    stages = f.stage_times()
    kernels = f.kernel_times()
    f.set_profiling(False)
    y = yd.cpu().numpy().astype(np.complex128)
    import oracle as O
    from oracle import fast
    rows = sampled_rows(N, a.rows, c.rows_seed)
    err, t_or = None, None
    if not a.no_oracle:
        el = O.element_geometry(V, F)
        t0 = time.perf_counter()
        yo = fast.matvec_rows(el, rows, x, c.k, c.alpha)
        t_or = time.perf_counter() - t0
        err = float(np.linalg.norm(y[rows] - yo) / np.linalg.norm(yo))
    solve = None
    if a.solve:
        # bm_solve (GMRES, tol 1e-4) of the plane-wave system; parity where a dense
        # solve is infeasible: the oracle's rows A_S on the sampled
        # rows give the sampled residual ‖A_S u − b_S‖/‖b_S‖ of the GPU solution;
        # the rigid-sphere series is a discretisation sanity check only
        el = O.element_geometry(V, F)
        b = O.plane_wave_rhs(el.centroid, el.normal, c.k, c.alpha, c.direction)
        u, info = f.solve(b, tol=c.gmres_tol, max_iter=a.max_iter, restart=a.restart, check=False)
        solve = {"tol": c.gmres_tol, **info}
        if not a.no_oracle:
            Au = fast.matvec_rows(el, rows, u, c.k, c.alpha)
            solve["sampled_residual"] = float(np.linalg.norm(Au - b[rows]) / np.linalg.norm(b[rows]))
            ser = O.rigid_sphere_total(el.centroid[rows], c.k, 0.5, c.direction)
            solve["rel_l2_vs_series_sampled"] = float(np.linalg.norm(u[rows] - ser) / np.linalg.norm(ser))
    print(json.dumps({"config": a.cfg, "N": N, "k": c.k, "mesh_s": round(t_mesh, 1), "build_s": round(t_build, 1),
                      "solve": solve,
                      "matvec_ms": round(mv_ms, 3), "stages_ms": {k: round(v, 3) for k, v in stages.items()},
                      "kernels_ms": {k: round(v, 3) for k, v in kernels.items()},
                      "sampled_rows": len(rows), "rel_l2_sampled": err, "oracle_rows_s": t_or, "tensor_cores": a.tc,
                      "lr_tensor_cores": a.lrtc, "alpha": str(c.alpha),
                      "oracle_cores": fast.num_threads(), "levels": levels,
                      "tree": {k: st[k] for k in ("n_levels", "n_hf_levels", "n_leaves", "n_m2l_pairs",
                                                  "n_direct_element_pairs", "n_corrections", "table_bytes",
                                                  "rank", "dirs")}}), flush=True)


if __name__ == "__main__":
    main()
