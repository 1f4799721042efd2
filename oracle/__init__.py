"""CPU oracle for arXiv 1208.3933 — TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper around ``oracle/oracle.c`` (plain single-threaded C that
follows Fig. 3 of the paper, line by line).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product package
``paper_1208_3933_b200`` never imports it and shares no code with it.

Parity status per function (DESIGN.md §4 lists the pins):
  makespan        pinned (SPEC worked example, brute force identities)
  johnson_order   pinned (brute force over all orders, SPEC example)
  Tables (PTM/LM/JM/QM/MM)  pinned (Table I sizes, closed forms, P3)
  lb / lb_eval    pinned for n <= 8 (P1 admissibility, P2 m=2 exactness,
                  P3 per-pair exactness, P4 leaves, P5 identical jobs,
                  P6 relabelling invariance, P7 envelope, P8 Table I counts);
                  large n: pinned only by transitivity (no printed LB values).
  bb_dfs          pinned (brute-force optimum n <= 8, Johnson for m = 2,
                  ta001 optimum 1278)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c with plain gcc -O2 (no SIMD intrinsics, no threads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC", "-o", _LIB, _SRC]
        )
    return _LIB


class _Tables(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("m", C.c_int32), ("P", C.c_int32),
        ("PTM", C.POINTER(C.c_int32)), ("MM", C.POINTER(C.c_int32)),
        ("LM", C.POINTER(C.c_int32)), ("JM", C.POINTER(C.c_int32)),
        ("QM", C.POINTER(C.c_int32)),
    ]


class _Counters(C.Structure):
    _fields_ = [(f, C.c_int64) for f in
                ("jm_reads", "lm_reads", "ptm_reads", "rm_reads", "qm_reads", "mm_reads")]


class _BBStats(C.Structure):
    _fields_ = [(f, C.c_int64) for f in ("bounded", "branched", "pruned", "leaves")]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        U16P = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
        _lib.ora_tables_build.argtypes = [I32P, C.c_int32, C.c_int32, C.POINTER(_Tables)]
        _lib.ora_tables_free.argtypes = [C.POINTER(_Tables)]
        _lib.ora_makespan.argtypes = [I32P, C.c_int32, C.c_int32, I32P, C.c_int32]
        _lib.ora_makespan.restype = C.c_int32
        _lib.ora_johnson_order.argtypes = [I32P, I32P, C.c_int32, I32P]
        _lib.ora_lb.argtypes = [C.POINTER(_Tables), U16P, C.c_int32,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.ora_lb.restype = C.c_int32
        _lib.ora_lb_eval.argtypes = [C.POINTER(_Tables), C.c_void_p, C.c_int32,
                                     C.c_void_p, C.c_int64, C.c_void_p]
        _lib.ora_bb_dfs.argtypes = [C.POINTER(_Tables), C.c_int32, C.c_int64,
                                    C.POINTER(C.c_int32), I32P, C.POINTER(_BBStats)]
    return _lib


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def makespan(ptm, perm) -> int:
    ptm = _i32(ptm)
    perm = _i32(perm)
    return int(lib().ora_makespan(ptm.ravel(), ptm.shape[0], ptm.shape[1], perm, len(perm)))


def johnson_order(a, b) -> np.ndarray:
    a, b = _i32(a), _i32(b)
    out = np.zeros(len(a), np.int32)
    lib().ora_johnson_order(a, b, len(a), out)
    return out


class Tables:
    """The six structures of §II-D for one instance."""

    def __init__(self, ptm):
        ptm = _i32(ptm)
        if ptm.ndim != 2:
            raise ValueError("ptm must be [n][m]")
        self.ptm = ptm
        self.n, self.m = ptm.shape
        self._t = _Tables()
        if lib().ora_tables_build(ptm.ravel(), self.n, self.m, C.byref(self._t)) != 0:
            raise ValueError("ora_tables_build rejected the instance")
        self.P = self._t.P

    def __del__(self):
        if getattr(self, "_t", None) is not None and _lib is not None:
            _lib.ora_tables_free(C.byref(self._t))
            self._t = None

    def _arr(self, name, rows, cols):
        ptr = getattr(self._t, name)
        return np.ctypeslib.as_array(ptr, shape=(rows * cols,)).reshape(rows, cols).copy()

    @property
    def MM(self):
        return self._arr("MM", self.P, 2)

    @property
    def LM(self):
        return self._arr("LM", self.n, self.P)

    @property
    def JM(self):
        return self._arr("JM", self.n, self.P)

    @property
    def QM(self):
        return self._arr("QM", self.n, self.m)

    def lb(self, prefix, detail: bool = False):
        """LB of one node (Fig. 3).  detail=True also returns per-couple values,
        the RM/QM minima and the Table I access counters."""
        pf = np.ascontiguousarray(prefix, dtype=np.uint16)
        if pf.size == 0:
            pf = np.zeros(1, np.uint16)
            d = 0
        else:
            d = len(prefix)
        if not detail:
            return int(lib().ora_lb(C.byref(self._t), pf, d, None, None, None, None))
        pv = np.zeros(self.P, np.int32)
        hd = np.zeros(self.m, np.int32)
        tl = np.zeros(self.m, np.int32)
        cnt = _Counters()
        v = lib().ora_lb(C.byref(self._t), pf, d, pv.ctypes.data, hd.ctypes.data,
                         tl.ctypes.data, C.addressof(cnt))
        counters = {f: getattr(cnt, f) for f, _ in _Counters._fields_}
        return int(v), pv, hd, tl, counters

    def lb_eval(self, prefix2d, depth) -> np.ndarray:
        """Batched LB with the fsp_lb_eval layout (host arrays)."""
        pf = np.ascontiguousarray(prefix2d, dtype=np.uint16)
        dp = _i32(depth)
        pool = dp.shape[0]
        stride = pf.shape[1] if pf.ndim == 2 else 0
        out = np.zeros(pool, np.int32)
        if pool == 0:
            return out
        rc = lib().ora_lb_eval(C.byref(self._t), pf.ctypes.data, stride, dp.ctypes.data,
                               pool, out.ctypes.data)
        if rc != 0:
            raise ValueError("malformed node in pool")
        return out

    def bb_dfs(self, initial_ub: int = 2**31 - 1, node_limit: int = 0):
        ms = C.c_int32(0)
        perm = np.zeros(self.n, np.int32)
        st = _BBStats()
        rc = lib().ora_bb_dfs(C.byref(self._t), int(initial_ub), int(node_limit),
                              C.byref(ms), perm, C.byref(st))
        if rc < 0:
            raise ValueError("ora_bb_dfs: bad arguments")
        stats = {f: getattr(st, f) for f, _ in _BBStats._fields_}
        return rc, int(ms.value), perm, stats
