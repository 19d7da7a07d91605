#!/usr/bin/env python
"""k_xlate_bf (opt.tensor_cores = 5) against the CUDA-core translations (tensor_cores = 0):
matvec difference and the tasks routed to each kernel family.

    python tools/xbf_check.py [--config 2] [--mesh 4]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from fda_inputs import config_mesh, CONFIGS, random_density, icosphere
    from paper_1403_4747_b200 import FDA
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=0)
    ap.add_argument("--mesh", type=int, default=4)
    ap.add_argument("--k", type=float, default=40.0)
    a = ap.parse_args()
    if a.config:
        c = CONFIGS[a.config]
        V, F = config_mesh(a.config)
        k, alpha, eps, ml = c.k, c.alpha, c.eps, c.max_leaf
    else:
        V, F = icosphere(a.mesh, 0.5)
        k, alpha, eps, ml = a.k, -1j / a.k, 1e-4, 32
    x = torch.from_numpy(random_density(len(F), 5).astype(np.complex64)).cuda()
    ys = {}
    for name, tc, kw, prof, mask in (("cuda_core", 0, {}, False, 7), ("xbf_graph", 5, {}, False, 7),
                                     ("xbf_serial", 5, {}, True, 7), ("xbf_m2m", 5, {}, False, 1),
                                     ("xbf_l2l", 5, {}, False, 2), ("xbf_m2l", 5, {}, False, 4),
                                     ("tc_default", 2, {}, False, 7)):
        os.environ["FDA_XBF_MASK"] = str(mask)
        f = FDA(V, F, k, alpha, eps, max_leaf=ml, tensor_cores=tc, **kw)
        if prof:
            f.set_profiling(True)
        y = f.matvec(x)
        torch.cuda.synchronize()
        y = f.matvec(x)          # second application (graph replay / warm path)
        torch.cuda.synchronize()
        ys[name] = y.cpu().numpy().astype(np.complex128)
        kt = {n: v for n, v in f.kernel_tasks().items() if v}
        e = np.linalg.norm(ys[name] - ys["cuda_core"]) / np.linalg.norm(ys["cuda_core"])
        print(json.dumps({"variant": name, "N": len(F), "rel_l2_vs_cuda_core": float(e), "kernel_tasks": kt}), flush=True)
        f.close()

if __name__ == "__main__":
    main()
