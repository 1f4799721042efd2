"""Thin ctypes binding of libfsp.so (include/fsp.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  Device buffers are torch CUDA tensors (PyTorch supplies memory
and streams); host buffers are numpy arrays.  There is no CPU fallback: if the
library is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# (FSP_LIB_VARIANT: diagnostics, a compile-time A/B build of the same library
# under paper_1208_3933_b200/_build/variants/, tools/build_variant.py)
LIB_PATH = os.path.join(_HERE, "libfsp.so") if not os.environ.get("FSP_LIB_VARIANT") else \
    os.path.join(_HERE, "_build", "variants", f"libfsp_{os.environ['FSP_LIB_VARIANT']}.so")

FSP_OK, FSP_EINVAL, FSP_ERANGE, FSP_ENOMEM, FSP_ECUDA = 0, -1, -2, -3, -4
FSP_ENOTFOUND, FSP_EBUDGET, FSP_EBADNODE = -5, -6, -7
_NAMES = {0: "FSP_OK", -1: "FSP_EINVAL", -2: "FSP_ERANGE", -3: "FSP_ENOMEM", -4: "FSP_ECUDA",
          -5: "FSP_ENOTFOUND", -6: "FSP_EBUDGET", -7: "FSP_EBADNODE"}

# every symbol include/fsp.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "fsp_instance_load", "fsp_instance_free", "fsp_instance_get_info", "fsp_lb_launch_info",
    "fsp_lb_eval", "fsp_lb_eval_children",
    "fsp_lb_eval_host", "fsp_lb_eval_sibling", "fsp_check", "fsp_lb_tune_pool", "fsp_lb_work", "fsp_bb_solve", "fsp_bb_solve_hybrid", "fsp_bb_init",
    "fsp_bb_step", "fsp_bb_ub_publish", "fsp_bb_ub_adopt", "fsp_bb_ub_get", "fsp_bb_ub_set",
    "fsp_bb_pool_size", "fsp_bb_node_bytes",
    "fsp_bb_export", "fsp_bb_import", "fsp_bb_debug_children", "fsp_bb_result", "fsp_bb_get_stats",
    "fsp_bb_free",
    "fsp_last_error", "fsp_version",
]


class FspError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


class InstanceInfo(C.Structure):
    _fields_ = [("n", C.c_int32), ("m", C.c_int32), ("P", C.c_int32), ("device", C.c_int32),
                ("groups", C.c_int32), ("pairs_per_group", C.c_int32),
                ("warps_per_cta", C.c_int32), ("ctas_per_sm", C.c_int32),
                ("smem_bytes", C.c_int32), ("maxm", C.c_int32), ("table_bytes", C.c_int64),
                ("nodes_per_lane", C.c_int32), ("walk16", C.c_int32)]


class LaunchInfo(C.Structure):
    _fields_ = [(f, C.c_int32) for f in (
        "grid", "warps_per_cta", "split", "iterations", "groups", "pairs_per_group",
        "group_buffers", "nodes_per_lane", "row_layout", "tmem_cols", "sparse_walk",
        "smem_bytes", "tail_split", "heads_jp", "mapping")]


class BBStats(C.Structure):
    _fields_ = [("bounded", C.c_int64), ("branched", C.c_int64), ("pruned", C.c_int64),
                ("leaves", C.c_int64), ("iterations", C.c_int64), ("wall_s", C.c_double),
                ("lb_ops", C.c_int64)]


_lib = None


def lib():
    """Load libfsp.so (raises if absent: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "fsp_instance_load": (C.c_int, [vp, i32, i32, C.POINTER(vp)]),
            "fsp_instance_free": (None, [vp]),
            "fsp_instance_get_info": (C.c_int, [vp, C.POINTER(InstanceInfo)]),
            "fsp_lb_launch_info": (C.c_int, [vp, i64, i32, C.POINTER(LaunchInfo)]),
            "fsp_lb_eval": (C.c_int, [vp, vp, i32, vp, i64, vp, vp]),
            "fsp_lb_eval_host": (C.c_int, [vp, vp, i32, vp, i64, vp]),
            "fsp_lb_eval_sibling": (C.c_int, [vp, vp, i32, vp, vp, i64, vp, vp]),
            "fsp_lb_eval_children": (C.c_int, [vp, vp, i32, vp, vp, i64, vp, vp]),
            "fsp_check": (C.c_int, [vp, vp]),
            "fsp_lb_tune_pool": (C.c_int, [vp, i32, C.c_double, C.POINTER(i64), vp, vp]),
            "fsp_lb_work": (i64, [i32, i32, i32]),
            "fsp_bb_solve": (C.c_int, [vp, i32, i64, C.c_double, C.POINTER(i32), vp,
                                       C.POINTER(BBStats)]),
            "fsp_bb_solve_hybrid": (C.c_int, [vp, i32, i32, i64, C.c_double, C.POINTER(i32), vp,
                                              C.POINTER(BBStats)]),
            "fsp_bb_init": (C.c_int, [vp, i32, i32, i32, C.POINTER(vp)]),
            "fsp_bb_step": (C.c_int, [vp, i32, vp]),
            "fsp_bb_ub_publish": (C.c_int, [vp, vp, vp]),
            "fsp_bb_ub_adopt": (C.c_int, [vp, vp, vp]),
            "fsp_bb_ub_get": (C.c_int, [vp, C.POINTER(i64)]),
            "fsp_bb_ub_set": (C.c_int, [vp, i64]),
            "fsp_bb_pool_size": (C.c_int, [vp, C.POINTER(i64)]),
            "fsp_bb_node_bytes": (i64, [vp]),
            "fsp_bb_export": (C.c_int, [vp, i64, vp, C.POINTER(i64)]),
            "fsp_bb_import": (C.c_int, [vp, vp, i64]),
            "fsp_bb_debug_children": (C.c_int, [vp, i64, vp, C.POINTER(i64)]),
            "fsp_bb_result": (C.c_int, [vp, C.POINTER(i32), vp]),
            "fsp_bb_get_stats": (C.c_int, [vp, C.POINTER(BBStats)]),
            "fsp_bb_free": (None, [vp]),
            "fsp_last_error": (C.c_char_p, []),
            "fsp_version": (C.c_int, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc, allow=()):
    if rc != FSP_OK and rc not in allow:
        raise FspError(rc, lib().fsp_last_error().decode())
    return rc


def _ptr(t):
    """Device pointer of a torch tensor (must be contiguous CUDA)."""
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def fsp_lb_work(n: int, m: int, d: int) -> int:
    return int(lib().fsp_lb_work(n, m, d))


class Instance:
    """An fsp_instance (tables resident on the current CUDA device)."""

    def __init__(self, ptm):
        ptm = np.ascontiguousarray(ptm, dtype=np.int32)
        if ptm.ndim != 2:
            raise ValueError("ptm must be [n][m]")
        self.n, self.m = ptm.shape
        self.ptm = ptm
        h = C.c_void_p()
        _check(lib().fsp_instance_load(ptm.ctypes.data, self.n, self.m, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().fsp_instance_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def info(self) -> dict:
        inf = InstanceInfo()
        _check(lib().fsp_instance_get_info(self._h, C.byref(inf)))
        return {f: getattr(inf, f) for f, _ in InstanceInfo._fields_}

    def launch_info(self, pool: int, sibling: bool = False) -> dict:
        """fsp_lb_launch_info: the bounding kernel's launch shape for a pool."""
        li = LaunchInfo()
        _check(lib().fsp_lb_launch_info(self._h, int(pool), int(bool(sibling)), C.byref(li)))
        return {f: getattr(li, f) for f, _ in LaunchInfo._fields_}

    def lb_eval(self, prefix, depth, out=None, stream=None):
        """fsp_lb_eval on torch CUDA tensors: prefix uint16-compatible
        [pool][stride] (torch.int16 storage), depth int32 [pool]."""
        import torch
        pool = depth.shape[0]
        if out is None:
            out = torch.empty(pool, dtype=torch.int32, device=depth.device)
        stride = prefix.shape[1] if prefix.dim() == 2 else 1
        _check(lib().fsp_lb_eval(self._h, _ptr(prefix), stride, _ptr(depth), pool, _ptr(out),
                                 _stream(stream)))
        return out

    def lb_eval_sibling(self, prefix, depth, completion=None, out=None, stream=None):
        """fsp_lb_eval_sibling on torch CUDA tensors (completion int32 [pool][m]
        or None)."""
        import torch
        pool = depth.shape[0]
        if out is None:
            out = torch.empty(pool, dtype=torch.int32, device=depth.device)
        stride = prefix.shape[1] if prefix.dim() == 2 else 1
        cp = _ptr(completion) if completion is not None else None
        _check(lib().fsp_lb_eval_sibling(self._h, _ptr(prefix), stride, _ptr(depth), cp, pool,
                                         _ptr(out), _stream(stream)))
        return out

    def lb_eval_children(self, prefix, depth, completion=None, out=None, stream=None):
        """fsp_lb_eval_children on torch CUDA tensors: out int32 [parents][32],
        out[p, t] = LB of parent p + its t-th unscheduled job (ascending)."""
        import torch
        B = depth.shape[0]
        if out is None:
            out = torch.full((B, 32), -1, dtype=torch.int32, device=depth.device)
        stride = prefix.shape[1] if prefix.dim() == 2 else 1
        cp = _ptr(completion) if completion is not None else None
        _check(lib().fsp_lb_eval_children(self._h, _ptr(prefix), stride, _ptr(depth), cp, B,
                                          _ptr(out), _stream(stream)))
        return out

    def lb_eval_host(self, prefix: np.ndarray, depth: np.ndarray, out=None):
        """fsp_lb_eval_host on numpy arrays (host memory, synchronous)."""
        prefix = np.ascontiguousarray(prefix, dtype=np.uint16)
        depth = np.ascontiguousarray(depth, dtype=np.int32)
        pool = depth.shape[0]
        if out is None:
            out = np.empty(pool, np.int32)
        stride = prefix.shape[1] if prefix.ndim == 2 else 1
        _check(lib().fsp_lb_eval_host(self._h, prefix.ctypes.data, stride, depth.ctypes.data,
                                      pool, out.ctypes.data))
        return out

    def lb_eval_host_ptr(self, prefix_ptr: int, stride: int, depth_ptr: int, pool: int,
                         out_ptr: int):
        """fsp_lb_eval_host on raw host pointers (e.g. pinned torch tensors)."""
        _check(lib().fsp_lb_eval_host(self._h, C.c_void_p(prefix_ptr), stride,
                                      C.c_void_p(depth_ptr), pool, C.c_void_p(out_ptr)))

    def tune_pool(self, max_log2: int = 22, frac: float = 0.95, stream=None):
        """fsp_lb_tune_pool: (chosen pool size, {size: bounds/s})."""
        pool = C.c_int64(0)
        rates = np.zeros(max_log2 - 11, np.float64)
        _check(lib().fsp_lb_tune_pool(self._h, int(max_log2), float(frac), C.byref(pool),
                                      rates.ctypes.data, _stream(stream)))
        return int(pool.value), {1 << (12 + i): float(r) for i, r in enumerate(rates)}

    def check(self, stream=None) -> int:
        """fsp_check: FSP_OK or FSP_EBADNODE (raises on other errors)."""
        return _check(lib().fsp_check(self._h, _stream(stream)), allow=(FSP_EBADNODE,))

    def bb_solve(self, initial_ub: int = 2**31 - 1, max_nodes: int = 0, time_limit_s: float = 0.0):
        """fsp_bb_solve.  Returns (status, makespan, perm, stats)."""
        ms = C.c_int32(0)
        perm = np.zeros(self.n, np.int32)
        st = BBStats()
        rc = lib().fsp_bb_solve(self._h, int(initial_ub), int(max_nodes), float(time_limit_s),
                                C.byref(ms), perm.ctypes.data, C.byref(st))
        _check(rc, allow=(FSP_ENOTFOUND, FSP_EBUDGET))
        return rc, int(ms.value), perm, {f: getattr(st, f) for f, _ in BBStats._fields_}

    def bb_solve_hybrid(self, threads: int = 4, initial_ub: int = 2**31 - 1, max_nodes: int = 0,
                        time_limit_s: float = 0.0):
        """fsp_bb_solve_hybrid.  Returns (status, makespan, perm, stats)."""
        ms = C.c_int32(0)
        perm = np.zeros(self.n, np.int32)
        st = BBStats()
        rc = lib().fsp_bb_solve_hybrid(self._h, int(initial_ub), int(threads), int(max_nodes),
                                       float(time_limit_s), C.byref(ms), perm.ctypes.data,
                                       C.byref(st))
        _check(rc, allow=(FSP_ENOTFOUND, FSP_EBUDGET))
        return rc, int(ms.value), perm, {f: getattr(st, f) for f, _ in BBStats._fields_}


class BBState:
    """Step-level device B&B (fsp_bb_init / fsp_bb_step / ...) for one rank."""

    def __init__(self, inst: Instance, initial_ub: int = 2**31 - 1, rank: int = 0, world: int = 1):
        self.inst = inst
        self.n = inst.n
        h = C.c_void_p()
        _check(lib().fsp_bb_init(inst._h, int(initial_ub), int(rank), int(world), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().fsp_bb_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, iters: int = 1, stream=None):
        _check(lib().fsp_bb_step(self._h, int(iters), _stream(stream)))

    def pool_size(self) -> int:
        v = C.c_int64(0)
        _check(lib().fsp_bb_pool_size(self._h, C.byref(v)))
        return int(v.value)

    def ub_publish(self, d_word) -> None:
        """(incumbent << 32) | rank -> a torch int64 CUDA tensor of one element."""
        _check(lib().fsp_bb_ub_publish(self._h, _ptr(d_word), _stream(None)))

    def ub_adopt(self, d_word) -> None:
        _check(lib().fsp_bb_ub_adopt(self._h, _ptr(d_word), _stream(None)))

    def ub_get(self) -> int:
        v = C.c_int64(0)
        _check(lib().fsp_bb_ub_get(self._h, C.byref(v)))
        return int(v.value)

    def ub_set(self, packed: int) -> None:
        _check(lib().fsp_bb_ub_set(self._h, int(packed)))

    def node_bytes(self) -> int:
        return int(lib().fsp_bb_node_bytes(self._h))

    def export(self, max_nodes: int, d_buf_ptr: int) -> int:
        k = C.c_int64(0)
        _check(lib().fsp_bb_export(self._h, int(max_nodes), C.c_void_p(d_buf_ptr), C.byref(k)))
        return int(k.value)

    def import_(self, d_buf_ptr: int, k: int):
        _check(lib().fsp_bb_import(self._h, C.c_void_p(d_buf_ptr), int(k)))

    def debug_children(self, max_nodes: int = 1 << 30):
        """The last iteration's child pool (test hook): (prefix u16 [k][stride],
        depth [k], completion times [k][m], LB [k]) as numpy arrays."""
        m, stride = self.inst.m, (self.n + 7) & ~7
        k = C.c_int64(0)
        _check(lib().fsp_bb_debug_children(self._h, 0, None, C.byref(k)))
        cap = min(int(max_nodes), int(k.value))
        buf = np.zeros(max(1, cap) * (stride * 2 + 8 + 4 * m), np.uint8)
        _check(lib().fsp_bb_debug_children(self._h, cap, buf.ctypes.data, C.byref(k)))
        k = int(k.value)
        o = 0
        pf = buf[o:o + k * stride * 2].view(np.uint16).reshape(k, stride); o += k * stride * 2
        dp = buf[o:o + 4 * k].view(np.int32); o += 4 * k
        Cc = buf[o:o + 4 * k * m].view(np.int32).reshape(k, m); o += 4 * k * m
        lb = buf[o:o + 4 * k].view(np.int32)
        return pf.copy(), dp.copy(), Cc.copy(), lb.copy()

    def result(self):
        ms = C.c_int32(0)
        perm = np.zeros(self.n, np.int32)
        rc = _check(lib().fsp_bb_result(self._h, C.byref(ms), perm.ctypes.data),
                    allow=(FSP_ENOTFOUND,))
        return rc, int(ms.value), perm

    def stats(self) -> dict:
        st = BBStats()
        _check(lib().fsp_bb_get_stats(self._h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in BBStats._fields_}
