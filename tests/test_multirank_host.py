"""Multi-rank (sharded) FDA host logic with a real collective:
two gloo ranks on CPU, each builds its shard of the operator (host-only
tables), applies it in complex128 (tests/host_exec.py) and the partial y are
summed with torch.distributed.all_reduce — the same exchange the GPU path does
with NCCL.  The sum must equal the oracle operator to the FDA tolerance and
the owned leaf ranges must partition the tree."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    from host_exec import apply_tables
    from paper_1403_4747_b200 import FDA
    from fda_inputs import icosphere, random_density
    torch.set_num_threads(1)
    threads = max(1, (os.cpu_count() or 2) // world)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    V, F = icosphere(4, 0.5)
    k = 40.0
    f = FDA(V, F, k, 1j / k, 1e-4, device=-1, max_leaf=16, rank=rank, nranks=world, build_threads=threads)
    x = random_density(len(F), 11)
    y = apply_tables(f, x)
    t = torch.from_numpy(np.stack([y.real, y.imag]))
    dist.all_reduce(t)
    owned = torch.from_numpy(f.table("owned").astype(np.int64))
    allowned = [torch.zeros_like(owned) for _ in range(world)]
    dist.all_gather(allowned, owned)
    if rank == 0:
        np.save(out + ".y.npy", (t[0] + 1j * t[1]).numpy())
        np.save(out + ".own.npy", torch.stack(allowned).numpy())
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_matvec(tmp_path):
    import oracle as O
    from oracle import fast
    from fda_inputs import icosphere, random_density
    out = str(tmp_path / "r")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    y = np.load(out + ".y.npy")
    own = np.load(out + ".own.npy")
    # contiguous, disjoint, covering ownership
    assert own[0, 0] == 0 and own[0, 1] == own[1, 0] and own[0, 3] == own[1, 2] and own[1, 3] == 5120
    V, F = icosphere(4, 0.5)
    k = 40.0
    el = O.element_geometry(V, F)
    x = random_density(len(F), 11)
    yo = fast.matvec_rows(el, np.arange(len(F)), x, k, 1j / k)
    assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < 1e-3
