#!/usr/bin/env python
"""Benchmark of the B200 FDA Burton–Miller matvec (BASELINE.json metric:
"FDA Burton-Miller matvec ms and GMRES solve s vs N,kD; %FP32/HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl fda|reference]

A step = one fda_matvec (gather → near field ∥ S2M → M2M → M2L → L2L → L2T →
scatter) over device-resident inputs of the config-2
workload (BASELINE configs[1]: icosphere s=6, N = 81,920, kD = 50, ε = 1e-4,
leaf 64).  GMRES (row a9) and the build (row a0) are timed once and reported
under "solve" and "build_s".  Under torchrun (N > 1) the operator is sharded
over the ranks (leaves split by work; each rank's upward pass covers its own
elements, one grouped ncclSend/ncclRecv exchanges the partial outgoing states
other ranks' interaction lists need, one all-reduce of y — DESIGN.md §7):
strong scaling of one matvec, the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FDA Burton-Miller matvec ms and GMRES solve s vs N,kD; %FP32/HBM roofline"
FP32_FLOPS_PER_EVAL = 62        # FP32 flops (FFMA = 2) of one near-field kernel evaluation
# ncu --set full capture of one whole config-2 matvec (tools/gpu_ncu_full.sh → tools/ncu_summary.py):
# source of roofline.traffic (dram bytes read + written) for the dominant stage
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "r01_ncu_full_matvec_config2.json")
STAGE_KERNELS = {"near": ("k_near",), "m2l": ("k_m2l_lr",), "s2m": ("k_s2m",), "l2t": ("k_l2t",)}
SMS, FP32_LANES = 148, 128


def _peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        mp = {}
    hbm = mp.get("hbm_gbs", 6650.0)
    clk = mp.get("sm_max_mhz", 1965.0)
    fp32 = SMS * FP32_LANES * 2 * clk * 1e6 / 1e12    # TFLOP/s, derived from unit counts × max clock
    src = ("derived: 148 SMs x 128 FP32 lanes x 2 flops x the max SM clock "
           f"({clk:.0f} MHz, {'MEASURED_PEAKS.json' if 'sm_max_mhz' in mp else 'fallback'}); "
           f"HBM peak {'measured (MEASURED_PEAKS.json)' if 'hbm_gbs' in mp else 'fallback'}")
    return hbm, fp32, src


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--id={index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [ln.strip().split(",") for ln in open(self.f.name) if ln.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for nm, v in zip(names, r[4:8]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def _stage_work(f, N):
    """Algorithmic work per stage of one matvec."""
    st = f.stats()
    mats = f.table("mats").reshape(-1, 3)
    work = {}
    work["near"] = {"evals": 3 * st["n_direct_element_pairs"], "corr_entries": st["n_corrections"]}
    for stage in ("m2m", "m2l", "l2l"):
        ops = f.table(stage).reshape(-1, 4)
        rc = mats[ops[:, 3], 1] * mats[ops[:, 3], 2] if len(ops) else np.zeros(0)
        work[stage] = {"ops": int(len(ops)), "flops": float(8 * rc.sum()),
                       "launches": 3 * int(len(set(ops[:, 0].tolist()))) if len(ops) else 0}
    lr = f.table("m2l_lr").reshape(-1, 6)      # §4.2 factored ops: V̂ (r×T) then Û (T×r)
    if len(lr):
        rv = mats[lr[:, 3], 1] * mats[lr[:, 3], 2] + mats[lr[:, 4], 1] * mats[lr[:, 4], 2]
        work["m2l"]["ops"] += int(len(lr))
        work["m2l"]["flops"] += float(8 * rv.sum())
        work["m2l"]["launches"] = 3 if work["m2l"]["ops"] > len(lr) else 0
        work["m2l"]["launches"] += 6
    lS, lT = f.table("leaf_S"), f.table("leaf_T")
    for stage, ids in (("s2m", lS), ("l2t", lT)):
        ids = ids[ids >= 0]
        ent = float((mats[ids, 1] * mats[ids, 2]).sum()) if len(ids) else 0.0
        work[stage] = {"entries": ent, "bytes": 8.0 * ent + 16.0 * N, "flops": 8.0 * ent}
    return work


def _config(c, N, ws, args):
    """The workload description shared by both arms (the same matvec)."""
    return {"workload": f"config {c.cfg}: {c.name}, eps={c.eps}, leaf {c.max_leaf}, plane wave "
                        f"{[float(v) for v in np.round(c.direction, 4)]}",
            "N": N, "k": c.k, "alpha": "-i/k (the paper's i/k, reading C25)", "eps": c.eps, "l2_flush": "256 MB write between steps",
            "tensor_cores": args.tensor_cores, "m2l_lowrank": bool(args.m2l_lowrank),
            "parallelism": (f"octree-sharded x{ws} (partial upward pass, NCCL exchange of outgoing states, "
                            f"all-reduce of y)") if ws > 1 else "single GPU"}


def _traffic(stage):
    """DRAM bytes (read + write) of one matvec's launches of `stage` from the
    committed ncu summary, or None when the stage's kernels are not uniquely named."""
    names = STAGE_KERNELS.get(stage)
    try:
        launches = json.load(open(PROFILE_SUMMARY))["launches"]
    except Exception:
        return None
    if not names:
        return None
    tot = [l.get("traffic_B") for l in launches if any(n in l["kernel"] for n in names)]
    return float(sum(tot)) if tot and None not in tot else None


def run_fda(args):
    import torch
    import torch.distributed as dist
    from fda_inputs import config_mesh, CONFIGS, random_density
    from paper_1403_4747_b200 import FDA

    ws, rank, local = _dist()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    c = CONFIGS[args.config]
    V, F = config_mesh(args.config)
    N = len(F)
    t0 = time.perf_counter()
    if ws > 1:
        # sharded operator: NCCL exchange of partial outgoing states + all-reduce of y
        threads = max(1, (os.cpu_count() or ws) // ws)
        f = FDA(V, F, c.k, c.alpha, c.eps, device=local, max_leaf=c.max_leaf, rank=rank, nranks=ws,
                build_threads=threads, tensor_cores=args.tensor_cores, m2l_lowrank=args.m2l_lowrank)
        f.comm_init()
    else:
        f = FDA(V, F, c.k, c.alpha, c.eps, device=local, max_leaf=c.max_leaf, tensor_cores=args.tensor_cores,
                m2l_lowrank=args.m2l_lowrank)
    build_s = time.perf_counter() - t0
    st = f.stats()
    x = torch.from_numpy(random_density(N, c.x_seed).astype(np.complex64)).to(dev)
    y = torch.empty_like(x)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        f.matvec(x, y)
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    clocks = Clocks(local) if rank == 0 or True else None
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize(dev)
    for i in range(args.steps):
        flush.zero_()
        starts[i].record(stream)
        f.matvec(x, y)
        ends[i].record(stream)
    torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    ck = clocks.stop() if clocks else None
    per = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = float(np.mean(per))
    if ws > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # per-stage device times (CUDA events on the launching streams), separate profiled pass
    f.set_profiling(True)
    acc = {}
    for i in range(max(3, min(args.steps, 10))):
        flush.zero_()
        f.matvec(x, y)
        torch.cuda.synchronize(dev)
        for kname, v in f.stage_times().items():
            acc.setdefault(kname, []).append(v)
    f.set_profiling(False)
    stage_ms = {kname: float(np.mean(v)) for kname, v in acc.items()}

    hbm, fp32, src = _peaks()
    work = _stage_work(f, N)
    stages = {}
    for sname, t in stage_ms.items():
        e = {"ms": round(t, 4)}
        w = work.get(sname)
        if sname == "near" and t > 0:
            ach = w["evals"] * FP32_FLOPS_PER_EVAL / (t * 1e-3) / 1e12
            e.update({"bound": "alu", "achieved": ach, "peak": fp32, "unit": "TFLOP/s", "frac": ach / fp32,
                      "evals_per_s": w["evals"] / (t * 1e-3)})
        elif sname in ("m2m", "m2l", "l2l") and t > 0 and w["flops"] > 0:
            ach = w["flops"] / (t * 1e-3) / 1e12
            e.update({"bound": "alu", "achieved": ach, "peak": fp32, "unit": "TFLOP/s", "frac": ach / fp32})
        elif sname in ("s2m", "l2t") and t > 0 and w["entries"] > 0:
            ach = w["bytes"] / (t * 1e-3) / 1e9
            e.update({"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm})
        stages[sname] = e
    # dominant kernel = k_near (the longest single launch of the matvec: ncu launch list in
    # profiles/); its duration measured live, inside the captured graph while the far field
    # runs concurrently, with CUDA events on its own stream (fda_near_time), L2 flushed
    near_live = []
    for i in range(max(3, min(args.steps, 50))):
        flush.zero_()
        f.matvec(x, y)
        near_live.append(f.near_time())
    t_near = float(np.mean(near_live))
    w = work["near"]
    ach = w["evals"] * FP32_FLOPS_PER_EVAL / (t_near * 1e-3) / 1e12
    roof = {"bound": "alu", "achieved": ach, "peak": fp32, "unit": "TFLOP/s", "frac": ach / fp32,
            "kernel": "k_near (near field S2T + corrections, row a7)", "ms_per_launch": round(t_near, 4),
            "timing": "live in the CUDA graph (concurrent with the far field), CUDA events on its stream",
            "traffic": _traffic("near") if args.config == 2 else None, "peak_source": src,
            "unit_of_work": f"{w['evals']} kernel evaluations x {FP32_FLOPS_PER_EVAL} flops"}
    launches = int(f.table("launches")[0])   # exact count of our kernels per matvec (engine.cu)

    # e2e: the C-ABI call with pinned HOST buffers (H2D + D2H inside the timed region)
    xh = torch.from_numpy(random_density(N, c.x_seed)).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    for _ in range(2):
        f.matvec(xh, yh)
    te = []
    for _ in range(args.steps):
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        f.matvec(xh, yh)
        te.append(time.perf_counter() - t1)
    e2e_ms = float(np.mean(te)) * 1e3

    # GMRES solve (row a9): plane wave, tol 1e-4, no restart; one untimed solve first
    # (allocates the cached Krylov workspace), then the timed one
    b = f.rhs_plane_wave(c.direction, device=True)
    torch.cuda.synchronize(dev)
    f.solve(b, tol=c.gmres_tol, max_iter=300, check=False)
    u, info = f.solve(b, tol=c.gmres_tol, max_iter=300, check=False)

    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "c64", "data": "synthetic",
            "config": _config(c, N, ws, args),
            "matvecs_per_s": round(1e3 / ms, 2),
            "roofline": roof,
            "stages": stages,
            "build_s": round(build_s, 3),
            "solve": {"iterations": info["iterations"], "s": round(info["t_solve_s"], 4),
                      "converged": info["converged"], "true_residual": info["true_residual"], "tol": c.gmres_tol},
            "tree": {"levels": st["n_levels"], "hf_levels": st["n_hf_levels"], "leaves": st["n_leaves"],
                     "m2l_pairs": st["n_m2l_pairs"], "direct_element_pairs": st["n_direct_element_pairs"],
                     "corrections": st["n_corrections"], "rank": st["rank"], "dirs": st["dirs"],
                     "table_bytes": st["table_bytes"]},
            "e2e": {"value": round(e2e_ms, 4), "unit": "ms", "h2d_bytes_per_step": 16 * N,
                    "d2h_bytes_per_step": 16 * N},
            "gpu_launches": launches * args.steps,
            "clocks": ck,
        }
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(c, V, F, rows=args.cpu_rows)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    f.close()
    return out


def cpu_baseline(c, V, F, rows: int):
    """The oracle (oracle/fast.py, plain C + numpy fp64), as it stands, on the
    host cores: a bounded sample of `rows` seeded rows of the same matvec,
    extrapolated to the full N."""
    import oracle as O
    from oracle import fast
    from fda_inputs import random_density, sampled_rows
    el = O.element_geometry(V, F)
    N = len(F)
    x = random_density(N, c.x_seed)
    r = sampled_rows(N, rows, c.rows_seed)
    fast.matvec_rows(el, r[:4], x, c.k, c.alpha)      # load/compile outside the timing
    t = time.perf_counter()
    fast.matvec_rows(el, r, x, c.k, c.alpha)
    dt = time.perf_counter() - t
    return {"value": round(dt * N / len(r) * 1e3, 2), "unit": "ms", "cores": fast.num_threads(), "kind": "oracle",
            "sample": f"{len(r)} seeded rows of the N={N} dense fp64 matvec ({dt:.2f} s), scaled by N/rows"}


def run_reference(args):
    """--impl reference: the oracle as it stands, timed on the host cores;
    each step = a bounded row sample, value = full-matvec ms extrapolated."""
    ws, rank, _ = _dist()
    if rank != 0:
        return None
    import oracle as O
    from oracle import fast
    from fda_inputs import config_mesh, CONFIGS, random_density, sampled_rows
    c = CONFIGS[args.config]
    V, F = config_mesh(args.config)
    N = len(F)
    el = O.element_geometry(V, F)
    x = random_density(N, c.x_seed)
    rows = sampled_rows(N, args.ref_rows * (args.steps + args.warmup), c.rows_seed)
    chunks = np.array_split(rows, args.steps + args.warmup)
    for i in range(args.warmup):
        fast.matvec_rows(el, chunks[i], x, c.k, c.alpha)
    ts = []
    for i in range(args.steps):
        r = chunks[args.warmup + i]
        t = time.perf_counter()
        fast.matvec_rows(el, r, x, c.k, c.alpha)
        ts.append((time.perf_counter() - t) * N / len(r) * 1e3)
    v = float(np.mean(ts))
    return {"impl": "reference", "metric": METRIC, "value": round(v, 2), "unit": "ms", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v, 2), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(c, N, ws, args),
            "cpu_baseline": {"value": round(v, 2), "unit": "ms", "cores": fast.num_threads(), "kind": "oracle",
                             "sample": f"{args.ref_rows} seeded rows per step of the N={N} dense fp64 matvec, "
                                       f"scaled by N/rows"},
            "e2e": {"value": round(v, 2), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="fda", choices=["fda", "reference"])
    ap.add_argument("--cpu-rows", type=int, default=1000)
    ap.add_argument("--ref-rows", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tensor-cores", type=int, default=2, help="dense translations on tcgen05 (3xTF32): 0 off, 1 all, 2 auto")
    ap.add_argument("--m2l-lowrank", type=int, default=1, help="§4.2 second-stage SVD of the M2L matrices")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    out = run_reference(args) if args.impl == "reference" else run_fda(args)
    if out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
