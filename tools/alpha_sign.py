"""GMRES iterations of the Burton–Miller system for α = +i/k and α = −i/k
(reading C1: kernel normal into the body) on one config: iterations, final
residual, and the solution against the rigid-sphere series on sampled rows.

    python tools/alpha_sign.py [--config 2] [--max-iter 400]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from fda_inputs import config_mesh, CONFIGS, sampled_rows
    from paper_1403_4747_b200 import FDA
    import oracle as O
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--max-iter", type=int, default=400)
    ap.add_argument("--tol", type=float, default=1e-4)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    V, F = config_mesh(a.config)
    el = O.element_geometry(V, F)
    rows = sampled_rows(len(F), 2000, c.rows_seed)
    ser = O.rigid_sphere_total(el.centroid[rows], c.k, 0.5, c.direction)
    for sgn in (+1, -1):
        alpha = sgn * 1j / c.k
        f = FDA(V, F, c.k, alpha, c.eps, max_leaf=c.max_leaf)
        b = f.rhs_plane_wave(c.direction)
        u, info = f.solve(b, tol=a.tol, max_iter=a.max_iter, check=False)
        err = float(np.linalg.norm(u[rows] - ser) / np.linalg.norm(ser))
        print(json.dumps({"config": a.config, "N": len(F), "k": c.k, "alpha": f"{'+' if sgn > 0 else '-'}i/k",
                          **info, "rel_l2_vs_series_sampled": err}), flush=True)
        f.close()


if __name__ == "__main__":
    main()
