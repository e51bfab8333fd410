"""ctypes front of the CPU oracle (oracle/oracle.cpp) -- TEST INFRASTRUCTURE.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(paper_2203_12878_b200) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.cpp")

STATUS = {0: "ok", 1: "parse", 2: "scope", 3: "barrier", 4: "range", 5: "arith", 8: "arg"}


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (-O2 -fopenmp); returns the .so path."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-shared", "-fPIC", "-o", _SO + ".tmp", _SRC]
        subprocess.run(cmd, check=True)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class _Res(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32), ("verdict", ctypes.c_int32),
        ("n_accesses", ctypes.c_uint64), ("n_racy_segments", ctypes.c_uint64),
        ("phase", ctypes.c_uint32), ("array", ctypes.c_uint32), ("block", ctypes.c_uint32),
        ("pad0", ctypes.c_uint32), ("index", ctypes.c_uint64),
        ("tid_lo", ctypes.c_uint32), ("tid_hi", ctypes.c_uint32),
        ("kind_lo", ctypes.c_uint32), ("kind_hi", ctypes.c_uint32),
        ("n_phases", ctypes.c_uint32), ("pad1", ctypes.c_uint32),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib.oracle_check.argtypes = [ctypes.c_char_p, u32p, u32p, ctypes.c_uint32,
                                     ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_uint64),
                                     ctypes.c_int, ctypes.POINTER(_Res), ctypes.c_char_p, ctypes.c_size_t]
        lib.oracle_check.restype = ctypes.c_int
        lib.oracle_enumerate.argtypes = [ctypes.c_char_p, u32p, u32p, ctypes.c_uint32,
                                         ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.c_int, ctypes.POINTER(ctypes.c_uint64), ctypes.c_uint64,
                                         ctypes.c_char_p, ctypes.c_size_t]
        lib.oracle_enumerate.restype = ctypes.c_int64
        lib.oracle_list_races.argtypes = lib.oracle_enumerate.argtypes
        lib.oracle_list_races.restype = ctypes.c_int64
        lib.oracle_arrays.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t]
        lib.oracle_arrays.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclass
class OracleResult:
    status: int
    verdict: int = 0
    n_accesses: int = 0
    n_racy_segments: int = 0
    witness: Optional[tuple] = None     # (phase, array, block, index, t_lo, t_hi, k_lo, k_hi)
    n_phases: int = 0
    diag: str = ""

    @property
    def racy(self) -> bool:
        return self.verdict == 1


def _args(grid, block, params):
    g = (ctypes.c_uint32 * 3)(*grid)
    b = (ctypes.c_uint32 * 3)(*block)
    names = list(params.keys())
    cn = (ctypes.c_char_p * max(1, len(names)))(*[n.encode() for n in names])
    cv = (ctypes.c_uint64 * max(1, len(names)))(*[int(params[n]) for n in names])
    return g, b, len(names), cn, cv


def check(src: str, grid: Sequence[int] = (1, 1, 1), block: Sequence[int] = (1, 1, 1),
          params: Optional[Dict[str, int]] = None, threads: int = 0) -> OracleResult:
    """Verdict, witness and access count of the MAP ``src`` at the instantiation."""
    lib = _load()
    params = params or {}
    g, b, n, cn, cv = _args(grid, block, params)
    res = _Res()
    diag = ctypes.create_string_buffer(512)
    nt = threads if threads > 0 else (os.cpu_count() or 1)
    lib.oracle_check(src.encode(), g, b, n, cn, cv, nt, ctypes.byref(res), diag, 512)
    out = OracleResult(status=res.status, diag=diag.value.decode(errors="replace"))
    if res.status == 0:
        out.verdict = res.verdict
        out.n_accesses = res.n_accesses
        out.n_racy_segments = res.n_racy_segments
        out.n_phases = res.n_phases
        if res.verdict:
            out.witness = (res.phase, res.array, res.block, res.index,
                           res.tid_lo, res.tid_hi, res.kind_lo, res.kind_hi)
    return out


def check_instance(inst, threads: int = 0) -> OracleResult:
    return check(inst.src, inst.grid, inst.block, inst.params, threads)


def enumerate_accesses(src: str, grid=(1, 1, 1), block=(1, 1, 1), params=None, threads: int = 1):
    """All emitted accesses as an (n, 6) uint64 array (phase, array, block, index, tid, kind)."""
    lib = _load()
    params = params or {}
    g, b, n, cn, cv = _args(grid, block, params)
    diag = ctypes.create_string_buffer(512)
    cnt = lib.oracle_enumerate(src.encode(), g, b, n, cn, cv, threads, None, 0, diag, 512)
    if cnt < 0:
        raise ValueError(f"oracle status {STATUS.get(-cnt, -cnt)}: {diag.value.decode()}")
    buf = np.zeros((max(cnt, 1), 6), dtype=np.uint64)
    lib.oracle_enumerate(src.encode(), g, b, n, cn, cv, threads,
                         buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), cnt, diag, 512)
    return buf[:cnt]


def list_races(src: str, grid=(1, 1, 1), block=(1, 1, 1), params=None, threads: int = 0):
    """Every racy segment's minimal pair (phase, array, block, index, t_lo, t_hi, k_lo, k_hi),
    in canonical order (the per-segment form of SPEC.md:434-437 races_of)."""
    lib = _load()
    params = params or {}
    g, b, n, cn, cv = _args(grid, block, params)
    diag = ctypes.create_string_buffer(512)
    nt = threads if threads > 0 else (os.cpu_count() or 1)
    cnt = lib.oracle_list_races(src.encode(), g, b, n, cn, cv, nt, None, 0, diag, 512)
    if cnt < 0:
        raise ValueError(f"oracle status {STATUS.get(-cnt, -cnt)}: {diag.value.decode()}")
    buf = np.zeros((max(cnt, 1), 8), dtype=np.uint64)
    lib.oracle_list_races(src.encode(), g, b, n, cn, cv, nt,
                          buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), cnt, diag, 512)
    return [tuple(int(x) for x in row) for row in buf[:cnt]]


def list_races_instance(inst, threads: int = 0):
    return list_races(inst.src, inst.grid, inst.block, inst.params, threads)


def array_names(src: str):
    lib = _load()
    buf = ctypes.create_string_buffer(4096)
    n = lib.oracle_arrays(src.encode(), buf, 4096)
    if n < 0:
        raise ValueError(buf.value.decode())
    return buf.value.decode().split("\n")[:n]
