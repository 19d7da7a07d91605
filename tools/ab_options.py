#!/usr/bin/env python
"""A/B of build options on the graph matvec time of a config (CUDA events, L2 flushed).

    python tools/ab_options.py --config 4 --variants '{}' '{"lr_tensor_cores": 1}' ...

A variant may carry "_env": {...} (environment set before its build).
One JSON line per variant: matvec ms (mean of --steps), per-kernel-family ms of a
profiled pass, relative difference of y against the first variant.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from fda_inputs import config_mesh, CONFIGS, random_density
    from paper_1403_4747_b200 import FDA
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--variants", nargs="+", default=["{}"])
    a = ap.parse_args()
    c = CONFIGS[a.config]
    V, F = config_mesh(a.config)
    x = torch.from_numpy(random_density(len(F), c.x_seed).astype(np.complex64)).cuda()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    y_ref = None
    prev_env = []
    for vs in a.variants:
        opts = json.loads(vs)
        env = opts.pop("_env", {})          # build-time environment knobs (engine experiments)
        for k in prev_env:
            os.environ.pop(k, None)
        os.environ.update({k: str(v) for k, v in env.items()})
        prev_env = list(env)
        f = FDA(V, F, c.k, c.alpha, c.eps, **opts)
        y = torch.empty_like(x)
        for _ in range(5):
            f.matvec(x, y)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f.matvec(x, y)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        near_live = f.near_time()
        f.set_profiling(True)
        f.matvec(x, y)
        torch.cuda.synchronize()
        kt = {k: round(v, 4) for k, v in f.kernel_times().items() if v > 0}
        f.set_profiling(False)
        yn = y.cpu().numpy().astype(np.complex128)
        if y_ref is None:
            y_ref = yn
        print(json.dumps({"config": a.config, "options": opts, "env": env, "near_live_ms": round(near_live, 4), "matvec_ms": round(float(np.mean(ts)), 4),
                          "kernels_ms": kt, "rel_vs_first": float(np.linalg.norm(yn - y_ref) / np.linalg.norm(y_ref)),
                          "build_s": round(f.stats()["t_build_s"], 2)}), flush=True)
        f.close()


if __name__ == "__main__":
    main()
