"""Multi-rank (sharded) FDA host logic with real collectives:
gloo ranks on CPU, each builds its shard of the operator (host-only tables)
and applies it in complex128 (tests/host_exec.py): partial upward pass on its
own elements, exchange of partial outgoing states with point-to-point
send/recv following the plan's xsend / xrecv lists (what the GPU path does
with grouped ncclSend/ncclRecv), downward pass for its own targets; the
partial y are summed with all_reduce.  The sum must equal the oracle operator
to the FDA tolerance, the owned leaf ranges must partition the tree, and
every rank's send list to a peer must be that peer's receive list."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# 1,280 elements at kD = 20: two HF levels (directional states cross the rank boundaries) and a
# host build of ≈ 10 s per single-threaded rank, so the 8-rank case stays within the CPU budget
MESH_SUBDIV, WAVENUMBER = 3, 20.0


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
    V, F = icosphere(MESH_SUBDIV, 0.5)
    k = WAVENUMBER
    f = FDA(V, F, k, 1j / k, 1e-4, device=-1, max_leaf=16, rank=rank, nranks=world, build_threads=threads)
    x = random_density(len(F), 11)
    xs_t, xr_t = f.table("xsend"), f.table("xrecv")

    def lists(tab):
        out, i = [], 0
        for _ in range(world):
            c = int(tab[i])
            out.append([int(v) for v in tab[i + 1:i + 1 + c]])
            i += 1 + c
        return out
    xsend, xrecv = lists(xs_t), lists(xr_t)
    oo = f.table("out_offset")
    lev = f.table("levels").reshape(-1, 4)
    boxes = f.table("boxes").reshape(-1, 8)
    outs = f.table("out_states").reshape(-1, 2)
    T = lambda s: int(lev[boxes[outs[s, 0], 0], 3])   # noqa: E731

    def exchange(ob):
        reqs, bufs = [], {}
        for q in range(world):
            if q == rank:
                continue
            if xsend[q]:
                pk = np.concatenate([ob[oo[s]:oo[s] + T(s)] for s in xsend[q]])
                reqs.append(dist.isend(torch.from_numpy(np.stack([pk.real, pk.imag])), dst=q))
            if xrecv[q]:
                n = sum(T(s) for s in xrecv[q])
                bufs[q] = torch.zeros(2, n, dtype=torch.float64)
                reqs.append(dist.irecv(bufs[q], src=q))
        for r in reqs:
            r.wait()
        for q, b in bufs.items():
            v = (b[0] + 1j * b[1]).numpy()
            o = 0
            for s in xrecv[q]:
                ob[oo[s]:oo[s] + T(s)] += v[o:o + T(s)]
                o += T(s)
    y = apply_tables(f, x, exchange=exchange)
    y_noex = apply_tables(f, x, near=False, corr=False) - apply_tables(f, x, near=False, corr=False, exchange=exchange)
    t = torch.from_numpy(np.stack([y.real, y.imag]))
    dist.all_reduce(t)
    t0 = torch.from_numpy(np.stack([y_noex.real, y_noex.imag]))
    dist.all_reduce(t0)
    plans = [None] * world
    dist.all_gather_object(plans, (xsend, xrecv))
    tb = [None] * world
    dist.all_gather_object(tb, int(f.stats()["table_bytes"]))
    owned = torch.from_numpy(f.table("owned").astype(np.int64))
    allowned = [torch.zeros_like(owned) for _ in range(world)]
    dist.all_gather(allowned, owned)
    if rank == 0:
        np.save(out + ".y.npy", (t[0] + 1j * t[1]).numpy())
        np.save(out + ".y_noex.npy", (t0[0] + 1j * t0[1]).numpy())
        np.save(out + ".own.npy", torch.stack(allowned).numpy())
        ok = all(plans[a][0][b] == plans[b][1][a] for a in range(world) for b in range(world) if a != b)
        np.save(out + ".plan_ok.npy", np.array([ok, sum(len(v) for p in plans for v in p[0])]))
        np.save(out + ".tb.npy", np.array(tb))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [3, 8])
def test_gloo_sharded_matvec(tmp_path, world):
    import oracle as O
    from oracle import fast
    from fda_inputs import icosphere, random_density
    out = str(tmp_path / "r")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    y = np.load(out + ".y.npy")
    y_noex = np.load(out + ".y_noex.npy")
    own = np.load(out + ".own.npy")
    ok, nsent = np.load(out + ".plan_ok.npy")
    assert ok and nsent > 0
    # contiguous, disjoint, covering ownership
    V, F = icosphere(MESH_SUBDIV, 0.5)
    assert own[0, 0] == 0 and own[0, 2] == 0 and own[-1, 3] == len(F)
    for r in range(world - 1):
        assert own[r, 1] == own[r + 1, 0] and own[r, 3] == own[r + 1, 2]
    k = WAVENUMBER
    el = O.element_geometry(V, F)
    x = random_density(len(F), 11)
    yo = fast.matvec_rows(el, np.arange(len(F)), x, k, 1j / k)
    assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < 1e-3
    # the exchange is needed: without it the far field changes by O(1)
    assert np.linalg.norm(y_noex) / np.linalg.norm(yo) > 1e-2
    # each rank built only its share of the operator tables (partition.cpp: needed matrices,
    # own correction rows).  On this small mesh the K̃ of the HF levels, which every rank
    # needs, dominate (measured 0.71-0.82 at 3 ranks, 0.43-0.53 at 8); at config 3 the
    # shards are 0.32-0.34 at 8 ranks (tests/test_gpu_parity.py)
    from paper_1403_4747_b200 import FDA
    full = FDA(V, F, k, 1j / k, 1e-4, device=-1, max_leaf=16).stats()["table_bytes"]
    tb = np.load(out + ".tb.npy")
    print(f"world {world}: table bytes per rank / unsharded = {np.round(tb / full, 3).tolist()}")
    assert tb.max() < (0.95 if world == 3 else 0.7) * full
