#!/usr/bin/env python
"""Benchmark of the B200 FDA Burton–Miller matvec (BASELINE.json metric:
"FDA Burton-Miller matvec ms and GMRES solve s vs N,kD; %FP32/HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl fda|reference]

A step = one fda_matvec (gather → near field ∥ S2M → M2M → M2L → L2L → L2T →
scatter) over device-resident inputs.  Default
workload: config 4 (BASELINE configs[3]: graded prolate spheroid, N ≈ 1.3 M,
kD = 300, ε = 1e-4, leaf 64) — the largest BASELINE config with a one-GPU
point (config 5 is specified for 8 GPUs).  Configs 2 and 3 are measured in
the same run under "other_configs" (matvec ms, kernel shares); config 5 with
--with-config5.  GMRES (row a9) and the build (row a0) are timed once and
reported under "solve" and "build_s".

--gpus N > 1 outside torchrun re-executes this script under
torch.distributed.run with N ranks (NCCL_DEBUG=INFO); it fails loudly when
fewer than N GPUs are visible.  Under torchrun the operator is sharded over
the ranks (leaves split by work; each rank's upward pass covers its own
elements, one grouped ncclSend/ncclRecv exchanges the partial outgoing states
other ranks' interaction lists need, one all-reduce of y — DESIGN.md §7):
strong scaling of one matvec, the time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FDA Burton-Miller matvec ms and GMRES solve s vs N,kD; %FP32/HBM roofline"
# Near-field roofline unit.  SURVEY §8(d) asks for the %FP32 peak from the kernel's executed
# FFMA/FADD/FMUL counts.  One evaluation (target centroid × source quadrature point of
# ∂G/∂n_y + α∂²G/∂n_x∂n_y) executes, per target lane, 29.67 FP32-pipe instructions — SASS of
# k_near's inner loop (2 source elements × 3 points for a target pair): 82 FFMA2 + 64 FMUL2 +
# 26 FADD2 = 172 packed instructions per 6 evaluation pairs (28.67 per lane-evaluation) plus
# 1 FMUL.RZ (sincos range reduction) per lane, and 3 MUFU.  Each occupies one FMA-pipe lane
# slot, i.e. 2 flop-equivalents at the FFMA peak (148 SMs × 128 lanes × 2 × clock), so
# `frac` is the FMA-pipe utilisation of the kernel (ncu's own figure: 74% at config 4).  The
# survey's hand count of the evaluation as written (≈ 65 instructions ≈ 100 flop; the kernel
# removes work with the identities of DESIGN.md §5) is reported alongside as frac_survey_unit.
FP32_INSTR_PER_EVAL = 29.67
FLOPS_PER_EVAL = 2 * FP32_INSTR_PER_EVAL
FLOPS_PER_EVAL_SURVEY = 100
SMS, FP32_LANES = 148, 128
# B200_PROFILING.md nominal dense peaks: TF32 1.1 PFLOP/s vs BF16 2.25 PFLOP/s
TF32_OVER_BF16 = 1.1 / 2.25
KERNELS = ["k_gather", "k_near", "k_s2m", "k_xlate", "k_xlate_tc", "k_xlate_tcw", "k_m2l_lr", "k_m2l_tcw", "k_l2t",
           "k_scatter", "memset", "k_xlate_bf"]


def _peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        mp = {}
    hbm = mp.get("hbm_gbs", 6650.0)
    clk = mp.get("sm_max_mhz", 1965.0)
    fp32 = SMS * FP32_LANES * 2 * clk * 1e6 / 1e12    # TFLOP/s, derived from unit counts × max clock
    bf16 = mp.get("bf16_tflops", 2250.0)
    tf32x3 = bf16 * TF32_OVER_BF16 / 3.0               # 3xTF32: three TF32 MMA passes per fp32-accurate product
    bf16x3 = bf16 / 3.0                                # BF16x3: three BF16 MMA passes (hi·hi + hi·lo + lo·hi)
    ub = None
    try:
        rows = [json.loads(l) for l in open(os.path.join(ROOT, "profiles", "r01_ubench_ffma2.jsonl")) if l.strip()]
        ub = max(r["tflops"] for r in rows if r.get("test") in ("ffma", "ffma2"))
    except Exception:
        pass
    src = {"fp32": f"derived: 148 SMs x 128 FP32 lanes x 2 flops x {clk:.0f} MHz "
                   f"({'MEASURED_PEAKS.json sm_max_mhz' if 'sm_max_mhz' in mp else 'fallback clock'})",
           "fp32_measured_ubench_tflops": ub,
           "hbm": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in mp else "fallback 6650 GB/s",
           "tf32x3": f"MEASURED_PEAKS.json bf16_tflops ({bf16}) x nominal TF32/BF16 (1.1/2.25) / 3 passes",
           "bf16x3": f"MEASURED_PEAKS.json bf16_tflops ({bf16}) / 3 passes"}
    return hbm, fp32, {"tensor": tf32x3, "tensor_bf16": bf16x3}, src


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
    """Algorithmic work per stage of one matvec: flops (complex-equivalent,
    8·rows·cols per op) and bytes (8 B per matrix entry once + 8 B per source state entry
    read + 16 B per destination entry read-modify-written, per op)."""
    st = f.stats()
    mats = f.table("mats").reshape(-1, 3)
    work = {"near": {"evals": 3 * st["n_direct_element_pairs"], "corr_entries": st["n_corrections"]}}
    lr = f.table("m2l_lr").reshape(-1, 6)      # §4.2 factored ops: V̂ (r×T) then Û (T×r)
    for stage in ("m2m", "m2l", "l2l"):
        ops = f.table(stage).reshape(-1, 4)
        m = ops[:, 3] if len(ops) else np.zeros(0, dtype=np.int64)
        R, C = mats[m, 1].astype(float), mats[m, 2].astype(float)
        flops = float(8 * (R * C).sum())
        um = np.unique(m)
        byts = float((8 * C + 16 * R).sum() + 8 * (mats[um, 1] * mats[um, 2]).sum())
        if stage == "m2l" and len(lr):
            r, T = mats[lr[:, 3], 1].astype(float), mats[lr[:, 3], 2].astype(float)
            flops += float(16 * (r * T).sum())
            uv = np.unique(np.concatenate([lr[:, 3], lr[:, 4]]))
            byts += float((8 * T + 16 * T).sum() + 8 * (mats[uv, 1] * mats[uv, 2]).sum())
        work[stage] = {"ops": int(len(ops)) + (int(len(lr)) if stage == "m2l" else 0), "flops": flops, "bytes": byts}
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
            "config_index": c.cfg, "N": N, "k": c.k, "alpha": "-i/k (the paper's i/k, reading C25)", "eps": c.eps,
            "l2_flush": "256 MB write between timed steps (> 126 MB L2)",
            "tensor_cores": args.tensor_cores, "m2l_lowrank": bool(args.m2l_lowrank),
            "parallelism": (f"octree-sharded x{ws} (partial upward pass, NCCL exchange of outgoing states, "
                            f"all-reduce of y)") if ws > 1 else "single GPU"}


def _family_work(f, work):
    """Algorithmic work and roofline class of every kernel family (fda_kernel_times order)."""
    kf = f.kernel_flops()
    fam = {}
    fam["k_near"] = ("alu", work["near"]["evals"] * FLOPS_PER_EVAL,
                     f"{work['near']['evals']} kernel evaluations x {FP32_INSTR_PER_EVAL} executed FP32-pipe "
                     f"instructions (SASS count) x 2 flop-equivalents (FMA-pipe slot at the FFMA peak)")
    for k in ("k_xlate", "k_m2l_lr"):
        fl = sum(v for n, v in kf.items() if n.startswith(k + "/"))
        fam[k] = ("alu", fl, "complex-equivalent flops, 8·rows·cols per op (16·r·T per factored M2L op)")
    for k in ("k_xlate_tc", "k_xlate_tcw", "k_m2l_tcw"):
        fl = sum(v for n, v in kf.items() if n.startswith(k + "/"))
        if k == "k_m2l_tcw" and f.opt.m2l_bf16:
            fam[k] = ("tensor_bf16", fl, "complex-equivalent flops on tcgen05 BF16x3 (k_m2l_bf: 16·r·T per factored op)")
        else:
            fam[k] = ("tensor", fl, "complex-equivalent flops on tcgen05 3xTF32 (8·rows·cols per op)")
    fl = sum(v for n, v in kf.items() if n.startswith("k_xlate_bf/"))
    fam["k_xlate_bf"] = ("tensor_bf16", fl, "complex-equivalent flops on tcgen05 BF16x3 (k_xlate_bf: 8·rows·cols per op)")
    fam["k_s2m"] = ("hbm", work["s2m"]["bytes"], "8 B per stored S̃ entry + 16 B per element")
    fam["k_l2t"] = ("hbm", work["l2t"]["bytes"], "8 B per stored T̃ entry + 16 B per element")
    return fam


def _measure(f, x, dev, steps, warmup, flush, stream, torch, clocks_index=None):
    y = torch.empty_like(x)
    for _ in range(warmup):
        f.matvec(x, y)
    torch.cuda.synchronize(dev)
    ck = Clocks(clocks_index) if clocks_index is not None else None
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        starts[i].record(stream)
        f.matvec(x, y)
        ends[i].record(stream)
    torch.cuda.synchronize(dev)
    ckv = ck.stop() if ck else None
    per = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    return per, ckv, y


def run_config(cfg, args, ws, rank, local, primary):
    import torch
    import torch.distributed as dist
    from fda_inputs import config_mesh, CONFIGS, random_density
    from paper_1403_4747_b200 import FDA

    dev = torch.device(f"cuda:{local}")
    c = CONFIGS[cfg]
    V, F = config_mesh(cfg)
    N = len(F)
    t0 = time.perf_counter()
    kw = dict(device=local, max_leaf=c.max_leaf, tensor_cores=args.tensor_cores, m2l_lowrank=args.m2l_lowrank)
    if ws > 1:
        threads = max(1, (os.cpu_count() or ws) // ws)
        f = FDA(V, F, c.k, c.alpha, c.eps, rank=rank, nranks=ws, build_threads=threads, **kw)
        f.comm_init()
    else:
        f = FDA(V, F, c.k, c.alpha, c.eps, **kw)
    build_s = time.perf_counter() - t0
    st = f.stats()
    x = torch.from_numpy(random_density(N, c.x_seed).astype(np.complex64)).to(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    steps = args.steps if primary else min(args.steps, 30)
    if ws > 1:
        dist.barrier()
    per, ck, y = _measure(f, x, dev, steps, args.warmup, flush, stream, torch, local if primary else None)
    ms = float(np.mean(per))
    if ws > 1:
        dist.barrier()
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # near-field kernel duration live inside the captured graph (external event nodes on its
    # stream, concurrent with the far field), the same timed loop shape
    near_live = []
    for _ in range(max(3, min(steps, 50))):
        flush.zero_()
        f.matvec(x, y)
        near_live.append(f.near_time())
    t_near_live = float(np.mean(near_live))

    # profiled pass: every kernel serialised on one stream, CUDA events around every launch
    f.set_profiling(True)
    acc, kacc = {}, {}
    for _ in range(max(3, min(steps, 10))):
        flush.zero_()
        f.matvec(x, y)
        torch.cuda.synchronize(dev)
        for kname, v in f.stage_times().items():
            acc.setdefault(kname, []).append(v)
        if ws == 1:
            for kname, v in f.kernel_times().items():
                kacc.setdefault(kname, []).append(v)
    f.set_profiling(False)
    stage_ms = {k: float(np.mean(v)) for k, v in acc.items()}
    kern_ms = {k: float(np.mean(v)) for k, v in kacc.items()}

    hbm, fp32, tpk, psrc = _peaks()
    work = _stage_work(f, N)
    stages = {}
    for sname, t in stage_ms.items():
        e = {"ms": round(t, 4)}
        w = work.get(sname)
        if sname == "near" and t > 0:
            ach = w["evals"] * FLOPS_PER_EVAL / (t * 1e-3) / 1e12
            e.update({"bound": "alu", "achieved": ach, "peak": fp32, "unit": "TFLOP/s", "frac": ach / fp32,
                      "evals_per_s": w["evals"] / (t * 1e-3),
                      "frac_survey_unit": w["evals"] * FLOPS_PER_EVAL_SURVEY / (t * 1e-3) / 1e12 / fp32})
        elif sname in ("m2m", "m2l", "l2l") and t > 0 and w["flops"] > 0:
            ach = w["flops"] / (t * 1e-3) / 1e12
            e.update({"flops": w["flops"], "achieved_tflops": ach, "translation_gbs": w["bytes"] / (t * 1e-3) / 1e9,
                      "translation_frac_hbm": w["bytes"] / (t * 1e-3) / 1e9 / hbm, "algorithmic_bytes": w["bytes"]})
        elif sname in ("s2m", "l2t") and t > 0 and w["entries"] > 0:
            ach = w["bytes"] / (t * 1e-3) / 1e9
            e.update({"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm})
        stages[sname] = e

    roof, kernels = None, None
    if kern_ms:
        fam = _family_work(f, work)
        tot = sum(kern_ms.values())
        kernels = {}
        for k, t in kern_ms.items():
            e = {"ms": round(t, 4), "share": round(t / tot, 4) if tot > 0 else None}
            if k in fam and t > 0 and fam[k][1] > 0:
                bound, amount, unit = fam[k]
                if bound == "hbm":
                    a, p, u = amount / (t * 1e-3) / 1e9, hbm, "GB/s"
                else:
                    a, p, u = amount / (t * 1e-3) / 1e12, (fp32 if bound == "alu" else tpk[bound]), "TFLOP/s"
                e.update({"bound": bound, "achieved": a, "peak": p, "unit": u, "frac": a / p, "work": unit})
            kernels[k] = e
        dom = max((k for k in kern_ms if k in fam), key=lambda k: kern_ms[k])
        bound, amount, unit = fam[dom]
        if dom == "k_near":
            t_dom, timing = t_near_live, ("live in the CUDA graph of the timed loop (concurrent with the far field): "
                                          "external event nodes on the near stream, L2 flushed, mean of launches")
        else:
            t_dom, timing = kern_ms[dom], "profiled pass: the family's launches serialised on one stream, CUDA events"
        if bound == "hbm":
            a, p, u = amount / (t_dom * 1e-3) / 1e9, hbm, "GB/s"
        else:
            a, p, u = amount / (t_dom * 1e-3) / 1e12, (fp32 if bound == "alu" else tpk[bound]), "TFLOP/s"
        roof = {"bound": "alu" if bound == "alu" else ("tensor" if bound.startswith("tensor") else bound),
                "achieved": a, "peak": p, "unit": u, "frac": a / p,
                "traffic": _traffic(cfg, dom), "kernel": dom, "ms_per_matvec": round(t_dom, 4),
                "share_of_kernel_time": round(kern_ms[dom] / tot, 4), "timing": timing, "unit_of_work": unit,
                "peak_source": psrc["fp32"] if bound == "alu" else (psrc["hbm"] if bound == "hbm" else
                                                                  psrc["bf16x3" if bound == "tensor_bf16" else "tf32x3"]),
                "fp32_measured_ubench_tflops": psrc["fp32_measured_ubench_tflops"]}
        if dom == "k_near":
            roof["frac_survey_unit"] = work["near"]["evals"] * FLOPS_PER_EVAL_SURVEY / (t_dom * 1e-3) / 1e12 / fp32
    launches = int(f.table("launches")[0])   # exact count of our kernels per matvec (engine.cu)
    out = {"cfg": cfg, "N": N, "ms": ms, "per_step_ms": [round(p, 4) for p in per[:5]], "build_s": build_s,
           "stages": stages, "kernels": kernels, "roofline": roof, "launches": launches, "clocks": ck,
           "near_live_ms": round(t_near_live, 4),
           "tree": {"levels": st["n_levels"], "hf_levels": st["n_hf_levels"], "leaves": st["n_leaves"],
                    "m2l_pairs": st["n_m2l_pairs"], "direct_element_pairs": st["n_direct_element_pairs"],
                    "corrections": st["n_corrections"], "rank": st["rank"], "dirs": st["dirs"],
                    "table_bytes": st["table_bytes"]}}
    if primary:
        # e2e: the C-ABI call with pinned HOST buffers (H2D + D2H inside the timed region); the
        # host vectors are complex64 (FDA_HOST_C64), the precision the device computes in
        xh = torch.from_numpy(random_density(N, c.x_seed).astype(np.complex64)).pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        for _ in range(2):
            f.matvec(xh, yh)
        te = []
        for _ in range(steps):
            torch.cuda.synchronize(dev)
            t1 = time.perf_counter()
            f.matvec(xh, yh)
            te.append(time.perf_counter() - t1)
        out["e2e_ms"] = float(np.mean(te)) * 1e3
        # GMRES solve (row a9): plane wave, tol 1e-4, no restart; one untimed solve first
        # (allocates the cached Krylov workspace), then the timed one
        b = f.rhs_plane_wave(c.direction, device=True)
        torch.cuda.synchronize(dev)
        try:   # sharded contexts run GMRES on owned slices (all-reduced dots, all-gathered vectors)
            f.solve(b, tol=c.gmres_tol, max_iter=300, check=False)
            u, info = f.solve(b, tol=c.gmres_tol, max_iter=300, check=False)
            out["solve"] = {"iterations": info["iterations"], "s": round(info["t_solve_s"], 4),
                            "converged": info["converged"], "true_residual": info["true_residual"],
                            "tol": c.gmres_tol, "sharded": ws > 1}
        except Exception as e:   # keep the matvec line when only the solve fails
            out["solve"] = {"error": str(e)[:200]}
    f.close()
    return out


def _traffic(cfg, kernel):
    """DRAM bytes (read + written) per matvec of `kernel` from a committed `ncu --set full`
    capture of this config's matvec (profiles/*_ncu_full_matvec_config<cfg>.json), or None."""
    import glob
    best = None
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", f"*_ncu_full_matvec_config{cfg}.json"))):
        best = p
    if best is None:
        return None
    try:
        launches = json.load(open(best))["launches"]
    except Exception:
        return None
    tot = [l.get("traffic_B") for l in launches if l["kernel"].split("<")[0].split("(")[0].strip().endswith(kernel)]
    return {"bytes_per_matvec": float(sum(tot)), "source": os.path.relpath(best, ROOT)} if tot and None not in tot \
        else None


def run_fda(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = _dist()
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from fda_inputs import CONFIGS
    primary = run_config(args.config, args, ws, rank, local, True)
    others = {}
    if not args.no_other_configs and ws == 1:
        extra = [c for c in (2, 3) if c != args.config] + ([5] if args.with_config5 and args.config != 5 else [])
        for c in extra:
            o = run_config(c, args, ws, rank, local, False)
            others[f"config{c}"] = {"N": o["N"], "matvec_ms": round(o["ms"], 4), "build_s": round(o["build_s"], 2),
                                    "stages": o["stages"], "kernels": o["kernels"], "roofline": o["roofline"]}
    out = None
    if rank == 0:
        c = CONFIGS[args.config]
        ms = primary["ms"]
        out = {
            "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "c64", "data": "synthetic",
            "config": _config(c, primary["N"], ws, args),
            "matvecs_per_s": round(1e3 / ms, 2),
            "roofline": primary["roofline"],
            "kernels": primary["kernels"],
            "stages": primary["stages"],
            "build_s": round(primary["build_s"], 3),
            "solve": primary.get("solve"),
            "tree": primary["tree"],
            "e2e": {"value": round(primary["e2e_ms"], 4), "unit": "ms", "h2d_bytes_per_step": 8 * primary["N"],
                    "d2h_bytes_per_step": 8 * primary["N"],
                    "path": "fda_matvec(FDA_HOST | FDA_HOST_C64): pinned complex64 in, H2D + gather + graph + "
                            "scatter + D2H"},
            "gpu_launches": primary["launches"] * args.steps,
            "clocks": primary["clocks"],
            "other_configs": others,
        }
        if not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(c)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def _oracle_rate_rows(N, budget_pairs):
    return max(2, int(budget_pairs // max(N, 1)))


def cpu_baseline(c):
    """The oracle (oracle/fast.py, plain C + numpy fp64), as it stands, on the
    host cores: a bounded sample of seeded rows of the same matvec (≈ 3e8
    element-pair evaluations, 10-30 s), extrapolated to the full N."""
    import oracle as O
    from oracle import fast
    from fda_inputs import config_mesh, random_density, sampled_rows
    V, F = config_mesh(c.cfg)
    el = O.element_geometry(V, F)
    N = len(F)
    x = random_density(N, c.x_seed)
    r = sampled_rows(N, min(N, _oracle_rate_rows(N, 3e8)), c.rows_seed)
    fast.matvec_rows(el, r[:2], x, c.k, c.alpha)      # load/compile outside the timing
    t = time.perf_counter()
    fast.matvec_rows(el, r, x, c.k, c.alpha)
    dt = time.perf_counter() - t
    return {"value": round(dt * N / len(r) * 1e3, 2), "unit": "ms", "cores": fast.num_threads(), "kind": "oracle",
            "sample": f"{len(r)} seeded rows of the N={N} dense fp64 matvec ({dt:.2f} s), scaled by N/rows"}


def run_reference(args):
    """--impl reference: the oracle as it stands, timed on the host cores;
    each step = a bounded row sample (the whole run ≈ 2.4e9 element-pair
    evaluations), value = full-matvec ms extrapolated."""
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
    per_step = min(N, _oracle_rate_rows(N, 2.4e9 / (args.steps + args.warmup)))
    rows = sampled_rows(N, min(N, per_step * (args.steps + args.warmup)), c.rows_seed)
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

    class A:
        tensor_cores, m2l_lowrank = args.tensor_cores, args.m2l_lowrank
    return {"impl": "reference", "metric": METRIC, "value": round(v, 2), "unit": "ms", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v, 2), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(c, N, ws, A),
            "cpu_baseline": {"value": round(v, 2), "unit": "ms", "cores": fast.num_threads(), "kind": "oracle",
                             "sample": f"{per_step} seeded rows per step of the N={N} dense fp64 matvec, "
                                       f"scaled by N/rows"},
            "e2e": {"value": round(v, 2), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _spawn(args):
    """--gpus N > 1 outside torchrun: re-execute under torch.distributed.run, one rank per GPU."""
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} requested but only {n} CUDA device(s) are visible\n")
        sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd, env=env))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="fda", choices=["fda", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true", help="skip the configs 2/3 lines")
    ap.add_argument("--with-config5", action="store_true", help="also measure config 5 (≈ 5 min build)")
    ap.add_argument("--tensor-cores", type=int, default=2, help="dense translations on tcgen05 (3xTF32): 0 off, 1 all, 2 auto")
    ap.add_argument("--m2l-lowrank", type=int, default=1, help="§4.2 second-stage SVD of the M2L matrices")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws, _, _ = _dist()
    if args.impl == "reference":          # the oracle on the host cores: rank 0 only, no GPU
        out = run_reference(args)
    else:
        if "WORLD_SIZE" in os.environ and ws != args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
            sys.exit(2)
        if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
            _spawn(args)
        out = run_fda(args)
    if out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
