"""PAPER.md §5.2 / Table 3 workload on one B200: a unit point
source at (-2, 0, 0) outside the rigid unit sphere, k = 5 and k = 50,
ε = 1e-3 (GMRES tol = ε), N = 106,580 (frequency-73 geodesic
sphere; the paper's mesh has 106,032).  The wideband-FMM comparison system is
out of scope; the paper's own T_it is printed beside ours as context.

    python tools/point_source.py [--nu 73]

One JSON line per k: build time, device matvec time, GMRES iterations and
time, relative L2 error of the solved surface potential against the
rigid-sphere point-source series (oracle/analytic.py, discretisation sanity).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PAPER_T_IT = {5.0: 2.15, 50.0: 12.38}   # Table 3, "Present", 1 Xeon core


def main():
    import torch
    import oracle as O
    from fda_inputs import POINT_SOURCE, point_source_mesh, bm_alpha
    from paper_1403_4747_b200 import FDA
    ap = argparse.ArgumentParser()
    ap.add_argument("--nu", type=int, default=POINT_SOURCE["nu"])
    a = ap.parse_args()
    V, F = point_source_mesh(a.nu, POINT_SOURCE["radius"])
    N = len(F)
    el = O.element_geometry(V, F)
    xs = POINT_SOURCE["source"]
    for k in POINT_SOURCE["ks"]:
        t0 = time.perf_counter()
        f = FDA(V, F, k, bm_alpha(k), POINT_SOURCE["eps"], max_leaf=POINT_SOURCE["max_leaf"])
        t_build = time.perf_counter() - t0
        b = f.rhs_point_source(xs, device=True)
        y = torch.empty_like(b)
        for _ in range(3):
            f.matvec(b, y)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            f.matvec(b, y)
        e.record()
        torch.cuda.synchronize()
        mv = s.elapsed_time(e) / 20
        u, info = f.solve(b, tol=POINT_SOURCE["gmres_tol"], max_iter=500, check=False)
        uh = u.cpu().numpy().astype(np.complex128)
        ser = O.rigid_sphere_point_source_total(el.centroid, k, POINT_SOURCE["radius"], xs)
        err = float(np.linalg.norm(uh - ser) / np.linalg.norm(ser))
        st = f.stats()
        print(json.dumps({"workload": "PAPER §5.2 point source (-2,0,0), unit sphere", "N": N, "k": k,
                          "eps": POINT_SOURCE["eps"], "build_s": round(t_build, 2), "matvec_ms": round(mv, 4),
                          "N_it": info["iterations"], "solve_s": round(info["t_solve_s"], 4),
                          "T_it_ms": round(info["t_solve_s"] / max(1, info["iterations"]) * 1e3, 3),
                          "converged": info["converged"], "true_residual": info["true_residual"],
                          "l2_error_vs_series": err, "levels": st["n_levels"], "hf_levels": st["n_hf_levels"],
                          "paper_T_it_s": PAPER_T_IT.get(k), "paper_N": 106032,
                          "paper_hardware": "1 core Xeon 5450"}), flush=True)
        f.close()


if __name__ == "__main__":
    main()
