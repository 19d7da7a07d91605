#!/usr/bin/env python
"""Reference solution u* of a BASELINE config, computed by the ORACLE only.

    python tools/oracle_solve.py --config 2 [--tol 1e-7] [--max-iter 80]

GMRES (oracle/solvers.py, §5, reading C20) on the dense
fp64 Burton–Miller operator of Eq. (5), every matvec evaluated row
by row by the plain-C oracle (oracle/fast.py → oracle/c/oracle_rows.c, all
host cores), right-hand side b = u_inc + α∂u_inc/∂n (oracle/analytic.py,
reading C22) for the config's plane wave.  Nothing here touches the CUDA
path: the output is a golden value for tests/test_gpu_parity.py
(test_config2_solution_vs_oracle_gmres), written to
tests/golden/config<C>_oracle_solution.npz with the GMRES history and the true
residual ‖b − A u*‖/‖b‖ of one extra oracle matvec.

Config 2 (N = 81,920) costs ≈ 256 s per oracle matvec on 8 cores.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from oracle import fast  # noqa: E402
from fda_inputs import config_mesh, CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--tol", type=float, default=1e-7)
    ap.add_argument("--max-iter", type=int, default=80)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    c = CONFIGS[args.config]
    V, F = config_mesh(args.config)
    el = O.element_geometry(V, F)
    N = len(F)
    rows = np.arange(N)
    b = O.plane_wave_rhs(el.centroid, el.normal, c.k, c.alpha, c.direction)
    count = [0]
    t0 = time.time()

    def matvec(x):
        y = fast.matvec_rows(el, rows, x, c.k, c.alpha)
        count[0] += 1
        print(f"[oracle_solve] matvec {count[0]} done at {time.time() - t0:.0f} s", flush=True)
        return y

    u, its, res, hist = O.gmres(matvec, b, tol=args.tol, max_iter=args.max_iter)
    true_res = float(np.linalg.norm(b - matvec(u)) / np.linalg.norm(b))
    out = args.out or os.path.join(ROOT, "tests", "golden", f"config{args.config}_oracle_solution.npz")
    meta = {"config": args.config, "N": N, "k": c.k, "alpha": [c.alpha.real, c.alpha.imag],
            "direction": [float(v) for v in c.direction], "tol": args.tol, "iterations": its,
            "gmres_residual": float(res), "true_residual": true_res, "history": [float(h) for h in hist],
            "threads": fast.num_threads(), "seconds": time.time() - t0,
            "source": "tools/oracle_solve.py: oracle.gmres on oracle.fast.matvec_rows (dense fp64 Eq. 5)"}
    np.savez_compressed(out, u=u.astype(np.complex128), meta=json.dumps(meta))
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
