#!/usr/bin/env python
"""Small end-to-end run for compute-sanitizer (one tool per gpurun call):

    compute-sanitizer --tool memcheck python tools/sanitize_small.py
    compute-sanitizer --tool racecheck python tools/sanitize_small.py

Exercises every kernel family on a 1,280-element mesh with HF levels: the device
build (k_e_*, k_zgemm, k_lowrank, k_corr), the near kernel (both CTA shapes
via two meshes), S2M / L2T, CUDA-core and tensor-core translations (k_xlate,
k_xlate_tc, k_xlate_tcw), the fused factored M2L (k_m2l_lr, k_m2l_tcw,
k_m2l_bf), the RHS pass, GMRES and the sharded halves with the one-GPU
exchange transport.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from fda_inputs import icosphere, random_density
    from paper_1403_4747_b200 import FDA, exchange_local
    V, F = icosphere(3, 0.5)
    k = 40.0
    x = random_density(len(F), 3)
    for opts in ({}, {"tensor_cores": 1, "lr_tensor_cores": 1}, {"tensor_cores": 4, "lr_tensor_cores": 1, "m2l_bf16": 0},
                 {"tensor_cores": 3, "m2l_lowrank": 0}):
        f = FDA(V, F, k, 1j / k, 1e-4, max_leaf=8, rhs_operator=1, **opts)
        y = f.matvec(x)
        b = f.rhs_apply(x)
        u, info = f.solve(f.rhs_plane_wave([0, 0, 1.0]), tol=1e-4, max_iter=50, check=False)
        print(opts, float(np.linalg.norm(y)), float(np.linalg.norm(b)), info["iterations"], flush=True)
        f.close()
    R = 2
    ranks = [FDA(V, F, k, 1j / k, 1e-4, max_leaf=8, rank=r, nranks=R, tensor_cores=1, lr_tensor_cores=1)
             for r in range(R)]
    xd = torch.from_numpy(x.astype(np.complex64)).cuda()
    ys = [torch.empty_like(xd) for _ in range(R)]
    for f, y in zip(ranks, ys):
        f.matvec_phase(xd, y, "up")
    torch.cuda.synchronize()
    exchange_local(ranks)
    for f, y in zip(ranks, ys):
        f.matvec_phase(xd, y, "down")
    torch.cuda.synchronize()
    print("sharded", float(sum(torch.linalg.norm(y).item() for y in ys)))
    print("SANITIZE_RUN_OK")


if __name__ == "__main__":
    main()
