"""Per-stage device times of the FDA matvec (profiling mode: stages serialised,
CUDA events, L2 flushed between matvecs).

    python tools/stage_times.py [--config 2] [--reps 20]
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
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tc", type=int, default=2, help="tcgen05 translations: 0 off, 1 all eligible, 2 auto")
    ap.add_argument("--lowrank", type=int, default=1, help="§4.2 second-stage SVD of K̃")
    a = ap.parse_args()
    c = CONFIGS[a.config]
    V, F = config_mesh(a.config)
    f = FDA(V, F, c.k, c.alpha, c.eps, max_leaf=c.max_leaf, tensor_cores=a.tc, m2l_lowrank=a.lowrank)
    x = torch.from_numpy(random_density(len(F), c.x_seed).astype(np.complex64)).cuda()
    y = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    f.matvec(x, y)
    f.set_profiling(True)
    acc = {}
    for _ in range(a.reps):
        flush.zero_()
        f.matvec(x, y)
        torch.cuda.synchronize()
        for k, v in f.stage_times().items():
            acc.setdefault(k, []).append(v)
    f.set_profiling(False)
    out = {k: round(float(np.median(v)), 4) for k, v in acc.items()}
    out["sum"] = round(sum(out.values()), 4)
    st = torch.cuda.Event(enable_timing=True)
    en = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(a.reps):
        flush.zero_()
        st.record()
        f.matvec(x, y)
        en.record()
        torch.cuda.synchronize()
        ts.append(st.elapsed_time(en))
    out["graph_matvec"] = round(float(np.median(ts)), 4)
    out["y_checksum"] = [float(y.real.sum()), float(y.imag.sum()), float(y.abs().sum())]
    print(json.dumps({"config": a.config, "tensor_cores": a.tc, "m2l_lowrank": a.lowrank,
                      "ms": out}))


if __name__ == "__main__":
    main()
