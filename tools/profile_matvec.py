"""Run W + K FDA matvecs of a config on cuda:0 (for ncu launch lists / captures).

    python tools/profile_matvec.py [--config 2] [--warmup 2] [--steps 3]
"""
import argparse
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
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--tc", type=int, default=2, help="tcgen05 translations: 0 off, 1 all eligible, 2 auto")
    a = ap.parse_args()
    c = CONFIGS[a.config]
    V, F = config_mesh(a.config)
    f = FDA(V, F, c.k, c.alpha, c.eps, max_leaf=c.max_leaf, tensor_cores=a.tc)
    x = torch.from_numpy(random_density(len(F), c.x_seed).astype(np.complex64)).cuda()
    y = torch.empty_like(x)
    for _ in range(a.warmup + a.steps):
        f.matvec(x, y)
    torch.cuda.synchronize()
    print("ok", f.stats()["n_m2l_pairs"], "launches_per_matvec", int(f.table("launches")[0]))


if __name__ == "__main__":
    main()
