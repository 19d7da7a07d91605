"""A/B of the factored-M2L kernels (opt.lr_tensor_cores 0 / 1 / 2) on one
config: the matvec of each mode against mode 0 (fused CUDA-core kernel),
profiled stage times and the graph matvec time.  One JSON line per mode.

    python tools/lrtc_check.py [--config 2] [--reps 20] [--modes 0,1,2]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(f, x, y, reps, flush):
    import torch
    f.matvec(x, y)
    f.set_profiling(True)
    acc = {}
    for _ in range(reps):
        flush.zero_()
        f.matvec(x, y)
        torch.cuda.synchronize()
        for k, v in f.stage_times().items():
            acc.setdefault(k, []).append(v)
    f.set_profiling(False)
    out = {k: round(float(np.median(v)), 4) for k, v in acc.items()}
    st = torch.cuda.Event(enable_timing=True)
    en = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        flush.zero_()
        st.record()
        f.matvec(x, y)
        en.record()
        torch.cuda.synchronize()
        ts.append(st.elapsed_time(en))
    out["graph_matvec"] = round(float(np.median(ts)), 4)
    return out


def main():
    import torch
    from fda_inputs import config_mesh, CONFIGS, random_density
    from paper_1403_4747_b200 import FDA
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--modes", default="0,1,2")
    a = ap.parse_args()
    c = CONFIGS[a.config]
    V, F = config_mesh(a.config)
    x = torch.from_numpy(random_density(len(F), c.x_seed).astype(np.complex64)).cuda()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    ref = None
    for m in [int(v) for v in a.modes.split(",")]:
        f = FDA(V, F, c.k, c.alpha, c.eps, max_leaf=c.max_leaf, lr_tensor_cores=m)
        y = torch.empty_like(x)
        ms = run(f, x, y, a.reps, flush)
        yn = y.cpu().numpy().astype(np.complex128)
        if ref is None:
            ref = yn
        d = float(np.linalg.norm(yn - ref) / np.linalg.norm(ref))
        print(json.dumps({"config": a.config, "lr_tensor_cores": m, "rel_vs_mode0": d, "ms": ms,
                          "launches": int(f.table("launches")[0])}), flush=True)
        f.close()


if __name__ == "__main__":
    main()
