"""Thin Python binding of libfda.so (include/fda.h): argument marshalling only.

Every step of the matvec, the right-hand side and the GMRES solve runs in the
library (host C++ build + sm_100a CUDA kernels); this module only converts
numpy / torch arguments to pointers.  It never falls back to Python or CPU
arithmetic: if the library cannot be loaded, or the context has no device,
the calls raise.

Host arrays are complex128 (numpy); device arrays are complex64 torch
tensors on the context's device.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfda.so")

FDA_HOST = 0
FDA_DEVICE = 1
FDA_LOCAL = 2
FDA_PHASE_UP = 4
FDA_PHASE_DOWN = 8
FDA_HOST_C64 = 16

STATUS = {0: "FDA_OK", 1: "FDA_E_INVALID_ARG", 2: "FDA_E_MESH", 3: "FDA_E_NOMEM", 4: "FDA_E_CUDA",
          5: "FDA_E_NCCL", 6: "FDA_E_NOT_CONVERGED", 7: "FDA_E_STATE", 8: "FDA_E_INTERNAL"}

# every symbol include/fda.h declares
EXPORTS = ["fda_options_default", "fda_build", "fda_matvec", "fda_rhs_plane_wave", "fda_rhs_point_source",
           "fda_rhs_apply", "bm_solve",
           "fda_stats", "fda_nccl_unique_id", "fda_comm_init", "fda_exchange_local",
           "fda_set_profiling", "fda_stage_times", "fda_kernel_times", "fda_near_time", "fda_debug_table",
           "fda_last_error", "fda_status_string", "fda_free"]

STAGES = ["gather", "near", "s2m", "m2m", "m2l", "l2l", "l2t", "scatter"]
KERNELS = ["k_gather", "k_near", "k_s2m", "k_xlate", "k_xlate_tc", "k_xlate_tcw", "k_m2l_lr", "k_m2l_tcw", "k_l2t",
           "k_scatter", "memset", "k_xlate_bf"]


class FdaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class fda_cplx(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class fda_options(ctypes.Structure):
    _fields_ = [("max_leaf", ctypes.c_int32), ("p_eq", ctypes.c_int32), ("p_chk_lf", ctypes.c_int32),
                ("p_chk_hf", ctypes.c_int32), ("eq_scale", ctypes.c_double), ("chk_scale_lf", ctypes.c_double),
                ("tier1_rho", ctypes.c_double), ("tier2_rho", ctypes.c_double), ("direct_all", ctypes.c_int32),
                ("device", ctypes.c_int32), ("build_threads", ctypes.c_int32), ("use_graph", ctypes.c_int32),
                ("verbose", ctypes.c_int32), ("m2l_lowrank", ctypes.c_int32),
                ("rhs_operator", ctypes.c_int32), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("tensor_cores", ctypes.c_int32), ("hf_leaves", ctypes.c_int32), ("lr_tensor_cores", ctypes.c_int32),
                ("build_on_device", ctypes.c_int32), ("m2l_bf16", ctypes.c_int32)]


class fda_solve_info(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32), ("rel_residual", ctypes.c_double),
                ("true_residual", ctypes.c_double), ("t_solve_s", ctypes.c_double)]


class fda_build_info(ctypes.Structure):
    _fields_ = [("n_elements", ctypes.c_int64), ("n_levels", ctypes.c_int32), ("n_hf_levels", ctypes.c_int32),
                ("n_boxes", ctypes.c_int64), ("n_leaves", ctypes.c_int64), ("n_out_states", ctypes.c_int64),
                ("n_in_states", ctypes.c_int64), ("n_m2l_pairs", ctypes.c_int64), ("n_m2m_ops", ctypes.c_int64),
                ("n_l2l_ops", ctypes.c_int64), ("n_direct_leaf_pairs", ctypes.c_int64),
                ("n_direct_element_pairs", ctypes.c_int64), ("n_corrections", ctypes.c_int64),
                ("n_matrices", ctypes.c_int64), ("table_bytes", ctypes.c_int64), ("t_build_s", ctypes.c_double),
                ("rank", ctypes.c_int32 * 32), ("dirs", ctypes.c_int32 * 32), ("width", ctypes.c_double * 32)]


_lib = None


def exchange_local(contexts) -> None:
    """fda_exchange_local: the one-GPU test transport of the sharded exchange
    (contexts = the FDA objects of ranks 0..n-1 of one sharded build)."""
    lib = load_library()
    arr = (ctypes.c_void_p * len(contexts))(*[c.ctx for c in contexts])
    st = lib.fda_exchange_local(arr, len(contexts))
    if st != 0:
        raise FdaError(st, (lib.fda_last_error(contexts[0].ctx) or b"").decode())


def load_library(path: str = LIB_PATH):
    """Load libfda.so (raises if it is missing — there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built: run `python -m paper_1403_4747_b200.build`")
    lib = ctypes.CDLL(path)
    vp, i32, i64, dp = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    lib.fda_options_default.argtypes = [ctypes.POINTER(fda_options)]
    lib.fda_build.argtypes = [vp, i64, vp, i64, dp, fda_cplx, dp, ctypes.POINTER(fda_options), ctypes.POINTER(vp)]
    lib.fda_matvec.argtypes = [vp, vp, vp, i32, vp]
    lib.fda_rhs_plane_wave.argtypes = [vp, ctypes.POINTER(ctypes.c_double * 3), vp, i32]
    lib.fda_rhs_point_source.argtypes = [vp, ctypes.POINTER(ctypes.c_double * 3), vp, i32]
    lib.fda_rhs_apply.argtypes = [vp, vp, vp, i32, vp]
    lib.bm_solve.argtypes = [vp, vp, vp, dp, i32, i32, ctypes.POINTER(fda_solve_info), i32]
    lib.fda_stats.argtypes = [vp, ctypes.POINTER(fda_build_info)]
    lib.fda_nccl_unique_id.argtypes = [vp]
    lib.fda_comm_init.argtypes = [vp, vp]
    lib.fda_exchange_local.argtypes = [ctypes.POINTER(vp), i32]
    lib.fda_set_profiling.argtypes = [vp, i32]
    lib.fda_near_time.argtypes = [vp, ctypes.POINTER(ctypes.c_double)]
    lib.fda_stage_times.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32)]
    lib.fda_kernel_times.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32)]
    lib.fda_debug_table.argtypes = [vp, ctypes.c_char_p, vp, ctypes.POINTER(i64), ctypes.POINTER(i32)]
    lib.fda_last_error.argtypes = [vp]
    lib.fda_last_error.restype = ctypes.c_char_p
    lib.fda_status_string.argtypes = [ctypes.c_int]
    lib.fda_status_string.restype = ctypes.c_char_p
    lib.fda_free.argtypes = [vp]
    lib.fda_free.restype = None
    for name in ("fda_options_default", "fda_build", "fda_matvec", "fda_rhs_plane_wave", "fda_rhs_point_source",
                 "fda_rhs_apply", "bm_solve",
                 "fda_stats", "fda_nccl_unique_id", "fda_comm_init", "fda_exchange_local", "fda_exchange_local",
                 "fda_set_profiling", "fda_stage_times", "fda_kernel_times", "fda_near_time", "fda_debug_table"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def default_options(**kw) -> fda_options:
    lib = load_library()
    o = fda_options()
    lib.fda_options_default(ctypes.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise AttributeError(k)
        setattr(o, k, v)
    return o


def _ptr_np(a: np.ndarray) -> int:
    return a.ctypes.data


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


class FDA:
    """One built FDA context: ``FDA(vertices, triangles, k, alpha, eps, **options)``."""

    def __init__(self, vertices, triangles, k: float, alpha: complex, eps: float = 1e-4, **options):
        self.lib = load_library()
        V = np.ascontiguousarray(vertices, dtype=np.float64)
        F = np.ascontiguousarray(triangles, dtype=np.int32)
        if V.ndim != 2 or V.shape[1] != 3 or F.ndim != 2 or F.shape[1] != 3:
            raise ValueError("vertices must be (nv,3) and triangles (nt,3)")
        self.opt = default_options(**options)
        self.n = F.shape[0]
        self.k = float(k)
        self.alpha = complex(alpha)
        ctx = ctypes.c_void_p()
        st = self.lib.fda_build(_ptr_np(V), V.shape[0], _ptr_np(F), F.shape[0], self.k,
                                fda_cplx(self.alpha.real, self.alpha.imag), float(eps), ctypes.byref(self.opt),
                                ctypes.byref(ctx))
        if st != 0:
            raise FdaError(st, self.lib.fda_last_error(None).decode())
        self.ctx = ctx
        self.device = self.opt.device

    # -- lifetime
    def close(self):
        if getattr(self, "ctx", None):
            self.lib.fda_free(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != 0:
            raise FdaError(st, self.lib.fda_last_error(self.ctx).decode())

    # -- calls
    def comm_init(self, group=None):
        """Sharded contexts (nranks > 1): create the library's NCCL communicator.
        The 128-byte NCCL id is made on rank 0 by the library and broadcast
        with torch.distributed (plumbing only)."""
        import torch
        import torch.distributed as dist
        buf = torch.zeros(128, dtype=torch.uint8)
        if self.opt.rank == 0:
            idb = (ctypes.c_uint8 * 128)()
            st = self.lib.fda_nccl_unique_id(ctypes.byref(idb))
            if st != 0:
                raise FdaError(st, self.lib.fda_last_error(None).decode())
            buf = torch.tensor(list(idb), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            b = buf.cuda()
            dist.broadcast(b, src=0, group=group)
            buf = b.cpu()
        else:
            dist.broadcast(buf, src=0, group=group)
        idb = (ctypes.c_uint8 * 128)(*buf.tolist())
        self._check(self.lib.fda_comm_init(self.ctx, ctypes.byref(idb)))

    def matvec(self, x, y=None, stream=None, local: bool = False):
        """y = A x.  numpy complex128 → numpy complex128 (host path), or torch
        complex64 CUDA tensors (device path, asynchronous on ``stream``).
        local=True (sharded contexts): this rank's rows only, no collective."""
        return self._apply(self.lib.fda_matvec, x, y, stream, FDA_LOCAL if local else 0)

    def matvec_phase(self, x, y, phase: str, kind: str = "lhs"):
        """One half of a sharded matvec around an external exchange ("up" or
        "down"; device tensors, this rank's rows only) — see fda_exchange_local."""
        flag = FDA_PHASE_UP if phase == "up" else FDA_PHASE_DOWN
        fn = self.lib.fda_matvec if kind == "lhs" else self.lib.fda_rhs_apply
        return self._apply(fn, x, y, None, FDA_LOCAL | flag)

    def rhs_apply(self, v, b=None, stream=None, local: bool = False):
        """b = B v, the right-hand-side operator of Eq. (4) (needs rhs_operator=1)."""
        return self._apply(self.lib.fda_rhs_apply, v, b, stream, FDA_LOCAL if local else 0)

    def _apply(self, fn, x, y=None, stream=None, extra: int = 0):
        if _is_torch(x) and not x.is_cuda:
            # host tensors (e.g. pinned complex128, or complex64 → FDA_HOST_C64): host path with raw pointers
            import torch
            if not (x.dtype in (torch.complex128, torch.complex64) and x.is_contiguous() and x.numel() == self.n):
                raise ValueError("host x must be a contiguous complex128 or complex64 tensor of length n")
            if y is None:
                y = torch.empty_like(x)
            if y.dtype != x.dtype:
                raise ValueError("host y must have the dtype of x")
            c64 = FDA_HOST_C64 if x.dtype == torch.complex64 else 0
            self._check(fn(self.ctx, x.data_ptr(), y.data_ptr(), FDA_HOST | c64 | extra, None))
            return y
        if _is_torch(x):
            import torch
            if not (x.is_cuda and x.dtype == torch.complex64 and x.is_contiguous() and x.numel() == self.n):
                raise ValueError("device x must be a contiguous complex64 CUDA tensor of length n")
            if y is None:
                y = torch.empty_like(x)
            s = stream.cuda_stream if stream is not None else torch.cuda.current_stream(x.device).cuda_stream
            self._check(fn(self.ctx, x.data_ptr(), y.data_ptr(), FDA_DEVICE | extra, s))
            return y
        xh = np.ascontiguousarray(x, dtype=np.complex128)
        if xh.shape != (self.n,):
            raise ValueError("x must have length n")
        yh = np.empty(self.n, dtype=np.complex128) if y is None else y
        self._check(fn(self.ctx, _ptr_np(xh), _ptr_np(yh), FDA_HOST | extra, None))
        return yh

    def rhs_plane_wave(self, direction, device: bool = False):
        d = (ctypes.c_double * 3)(*[float(v) for v in direction])
        if device:
            import torch
            b = torch.empty(self.n, dtype=torch.complex64, device=f"cuda:{self.device}")
            self._check(self.lib.fda_rhs_plane_wave(self.ctx, ctypes.byref(d), b.data_ptr(), FDA_DEVICE))
            return b
        b = np.empty(self.n, dtype=np.complex128)
        self._check(self.lib.fda_rhs_plane_wave(self.ctx, ctypes.byref(d), _ptr_np(b), FDA_HOST))
        return b

    def rhs_point_source(self, source, device: bool = False):
        """fda_rhs_point_source: BM right-hand side of a unit point source (§5.2)."""
        d = (ctypes.c_double * 3)(*[float(v) for v in source])
        if device:
            import torch
            b = torch.empty(self.n, dtype=torch.complex64, device=f"cuda:{self.device}")
            self._check(self.lib.fda_rhs_point_source(self.ctx, ctypes.byref(d), b.data_ptr(), FDA_DEVICE))
            return b
        b = np.empty(self.n, dtype=np.complex128)
        self._check(self.lib.fda_rhs_point_source(self.ctx, ctypes.byref(d), _ptr_np(b), FDA_HOST))
        return b

    def solve(self, rhs, tol: float = 1e-4, max_iter: int = 200, restart: int = 0, check: bool = True):
        """bm_solve: GMRES on the FDA operator.  Returns (u, info dict)."""
        info = fda_solve_info()
        if _is_torch(rhs):
            import torch
            u = torch.empty_like(rhs)
            st = self.lib.bm_solve(self.ctx, rhs.data_ptr(), u.data_ptr(), float(tol), int(max_iter), int(restart),
                                   ctypes.byref(info), FDA_DEVICE)
        else:
            b = np.ascontiguousarray(rhs, dtype=np.complex128)
            u = np.empty(self.n, dtype=np.complex128)
            st = self.lib.bm_solve(self.ctx, _ptr_np(b), _ptr_np(u), float(tol), int(max_iter), int(restart),
                                   ctypes.byref(info), FDA_HOST)
        if st not in (0, 6) or (check and st != 0):
            self._check(st)
        return u, {"iterations": info.iterations, "converged": bool(info.converged),
                   "rel_residual": info.rel_residual, "true_residual": info.true_residual,
                   "t_solve_s": info.t_solve_s}

    def stats(self) -> dict:
        bi = fda_build_info()
        self._check(self.lib.fda_stats(self.ctx, ctypes.byref(bi)))
        d = {name: getattr(bi, name) for name, _ in fda_build_info._fields_ if name not in ("rank", "dirs", "width")}
        nl = bi.n_levels
        d["rank"] = list(bi.rank)[:nl]
        d["dirs"] = list(bi.dirs)[:nl]
        d["width"] = list(bi.width)[:nl]
        return d

    def set_profiling(self, on: bool = True):
        self._check(self.lib.fda_set_profiling(self.ctx, 1 if on else 0))

    def near_time(self) -> float:
        """fda_near_time: ms of the near-field kernel in the last matvec (live, in the graph)."""
        ms = ctypes.c_double()
        self._check(self.lib.fda_near_time(self.ctx, ctypes.byref(ms)))
        return ms.value

    def stage_times(self) -> dict:
        ms = (ctypes.c_double * 8)()
        n = ctypes.c_int32(8)
        self._check(self.lib.fda_stage_times(self.ctx, ms, ctypes.byref(n)))
        return {STAGES[i]: ms[i] for i in range(n.value)}

    def kernel_times(self) -> dict:
        """fda_kernel_times: ms per kernel family of the last profiled device matvec."""
        ms = (ctypes.c_double * len(KERNELS))()
        n = ctypes.c_int32(len(KERNELS))
        self._check(self.lib.fda_kernel_times(self.ctx, ms, ctypes.byref(n)))
        return {KERNELS[i]: ms[i] for i in range(n.value)}

    _DTYPES = {"perm": np.int64, "verts": np.float64, "leaf_range": np.int64, "leaf_S": np.int64,
               "leaf_T": np.int64, "leaf_S_rhs": np.int64, "corr_ptr_rhs": np.int64, "corr_col_rhs": np.int64,
               "corr_val_rhs": np.complex64, "leaf_out": np.int64, "leaf_in": np.int64, "out_offset": np.int64,
               "in_offset": np.int64, "sizes": np.int64, "m2m": np.int64, "m2l": np.int64, "l2l": np.int64, "m2l_lr": np.int64,
               "mats": np.int64, "specs": np.int64, "pool": np.complex64, "near_ptr": np.int64,
               "near_idx": np.int64, "corr_ptr": np.int64, "corr_col": np.int64, "corr_val": np.complex64,
               "out_states": np.int64, "in_states": np.int64, "boxes": np.int64, "box_center": np.float64,
               "levels": np.float64, "root": np.float64, "launches": np.int64, "owned": np.int64,
               "xsend": np.int64, "xrecv": np.int64, "hf_s2m": np.int64, "hf_s2m_rhs": np.int64,
               "hf_l2t": np.int64, "kernel_tasks": np.int64, "kernel_flops": np.float64}

    KERNEL_FAMILIES = ("k_xlate", "k_xlate_tc", "k_xlate_tcw", "k_m2l_lr", "k_m2l_tcw", "k_xlate_bf")

    def kernel_tasks(self) -> dict:
        """CTA tasks per translation kernel family and stage ("k_xlate_tc/m2m", …):
        where the build routed the translations (fda_debug_table "kernel_tasks")."""
        t = self.table("kernel_tasks").reshape(len(self.KERNEL_FAMILIES), 3)
        return {f"{f}/{s}": int(t[i, j]) for i, f in enumerate(self.KERNEL_FAMILIES)
                for j, s in enumerate(("m2m", "m2l", "l2l"))}

    def kernel_flops(self) -> dict:
        """Algorithmic flops per translation kernel family and stage (complex-equivalent,
        8·rows·cols per op; 16·r·T per factored M2L op)."""
        t = self.table("kernel_flops").reshape(len(self.KERNEL_FAMILIES), 3)
        return {f"{f}/{s}": float(t[i, j]) for i, f in enumerate(self.KERNEL_FAMILIES)
                for j, s in enumerate(("m2m", "m2l", "l2l"))}

    def table(self, name: str) -> np.ndarray:
        """A host-side build table (host-logic tests only)."""
        cnt = ctypes.c_int64()
        eb = ctypes.c_int32()
        self._check(self.lib.fda_debug_table(self.ctx, name.encode(), None, ctypes.byref(cnt), ctypes.byref(eb)))
        out = np.empty(cnt.value, dtype=self._DTYPES[name])
        assert out.itemsize == eb.value, (name, out.itemsize, eb.value)
        self._check(self.lib.fda_debug_table(self.ctx, name.encode(), out.ctypes.data, ctypes.byref(cnt),
                                             ctypes.byref(eb)))
        return out
