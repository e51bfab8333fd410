"""paper_2203_12878_b200 -- B200-native concrete MAP data-race checker.

Thin ctypes binding of the C ABI in include/mapcheck.h (argument marshalling
only: every step of the hot path runs in the sm_100a kernels of
libmapcheck.so).  PyTorch supplies device memory (the scratch buffer) and the
CUDA stream.  There is no CPU fallback: if the library is missing, importing
this package raises; if there is no GPU, ``check_races`` raises MapError
(MAP_E_CUDA).

Paper: arxiv 2203.12878 -- a MAP instantiated at fixed
grid/block dims and parameters is enumerated exhaustively; two distinct threads
touching one index of one array in one barrier phase, one of them writing, is a
data race; by Theorem 1 the verdict is
the ground truth for a typable kernel at that instantiation.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmapcheck.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2203_12878_b200._build` "
        "(nvcc, sm_100a).  There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

STATUS = {
    0: "MAP_OK", 1: "MAP_E_PARSE", 2: "MAP_E_SCOPE", 3: "MAP_E_BARRIER", 4: "MAP_E_RANGE",
    5: "MAP_E_ARITH", 6: "MAP_E_CUDA", 7: "MAP_E_COMM", 8: "MAP_E_ARG", 9: "MAP_E_NOMEM", 10: "MAP_E_TYPE",
}

EXPORTS = (
    "map_compile", "map_info_get", "map_scratch_bytes", "map_check_races", "map_witness_get",
    "map_program_free", "map_status_str", "map_chunk_count", "map_generate_bucketed",
    "map_sort_detect", "map_unpack_witness", "map_array_name", "map_chunk_info", "map_list_races",
    "map_default_chunk", "map_rank_chunks", "map_infer",
)


class _Instance(ctypes.Structure):
    _fields_ = [("grid", ctypes.c_uint32 * 3), ("block", ctypes.c_uint32 * 3), ("n_params", ctypes.c_uint32),
                ("param_names", ctypes.POINTER(ctypes.c_char_p)), ("param_values", ctypes.POINTER(ctypes.c_uint64))]


KERNEL_CLASSES = ("generate", "hist", "scan", "onesweep", "detect", "other", "onesweep_next",
                  "direct", "clear", "unit")   # MAP_K_* order
_NK = len(KERNEL_CLASSES)


class _Stats(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_float * _NK), ("launches", ctypes.c_uint32 * _NK), ("bytes", ctypes.c_uint64 * _NK),
                ("timed", ctypes.c_uint32 * _NK)]


class _Exec(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("scratch", ctypes.c_void_p),
                ("scratch_bytes", ctypes.c_size_t), ("chunk_max_accesses", ctypes.c_uint64),
                ("rank", ctypes.c_uint32), ("world", ctypes.c_uint32), ("stats", ctypes.POINTER(_Stats)),
                ("flags", ctypes.c_uint32)]

GEN_PATHS = {"auto": 0, "vm": 1, "jit": 2}
DETECT_PATHS = {"auto": 0x00, "sort": 0x10, "table": 0x20, "direct": 0x40, "unit": 0x80}   # MAP_DETECT_* (mapcheck.h)
EXEC_SEQUENTIAL = 0x100                                                       # MAP_EXEC_SEQUENTIAL
EXEC_PROFILE_GENERATE = 0x200                                                 # MAP_EXEC_PROFILE_GENERATE
EXEC_PROFILE_SAMPLED = 0x400                                                  # MAP_EXEC_PROFILE_SAMPLED


class _Result(ctypes.Structure):
    _fields_ = [("verdict", ctypes.c_int32), ("n_chunks", ctypes.c_int32), ("n_accesses", ctypes.c_uint64),
                ("racy_segments", ctypes.c_uint64), ("device_ms", ctypes.c_float), ("gpu_launches", ctypes.c_uint32),
                ("h2d_bytes", ctypes.c_uint64), ("d2h_bytes", ctypes.c_uint64)]


class _Witness(ctypes.Structure):
    _fields_ = [("phase", ctypes.c_uint32), ("array", ctypes.c_uint32), ("block", ctypes.c_uint32),
                ("index", ctypes.c_uint64), ("tid_lo", ctypes.c_uint32), ("tid_hi", ctypes.c_uint32),
                ("kind_lo", ctypes.c_uint8), ("kind_hi", ctypes.c_uint8), ("array_name", ctypes.c_char_p)]


class _ChunkDesc(ctypes.Structure):
    _fields_ = [("phase_lo", ctypes.c_uint32), ("phase_hi", ctypes.c_uint32), ("block_lo", ctypes.c_uint32),
                ("block_hi", ctypes.c_uint32), ("bound", ctypes.c_uint64), ("sort_bits", ctypes.c_uint32),
                ("n_passes", ctypes.c_uint32)]


class _Info(ctypes.Structure):
    _fields_ = [("n_phases", ctypes.c_uint32), ("n_arrays", ctypes.c_uint32), ("n_instances", ctypes.c_uint32),
                ("n_groups", ctypes.c_uint32), ("max_accesses", ctypes.c_uint64),
                ("max_unit_accesses", ctypes.c_uint64), ("u32_mode", ctypes.c_uint32),
                ("bytecode_ops", ctypes.c_uint32)]


_P = ctypes.c_void_p
_lib.map_compile.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(_Instance), ctypes.POINTER(_P),
                             ctypes.c_char_p, ctypes.c_size_t]
_lib.map_compile.restype = ctypes.c_int
_lib.map_info_get.argtypes = [_P, ctypes.POINTER(_Info)]
_lib.map_info_get.restype = ctypes.c_int
_lib.map_scratch_bytes.argtypes = [_P, ctypes.c_uint64]
_lib.map_scratch_bytes.restype = ctypes.c_size_t
_lib.map_check_races.argtypes = [_P, ctypes.POINTER(_Exec), ctypes.POINTER(_Result)]
_lib.map_check_races.restype = ctypes.c_int
_lib.map_witness_get.argtypes = [_P, ctypes.POINTER(_Witness)]
_lib.map_witness_get.restype = ctypes.c_int
_lib.map_program_free.argtypes = [_P]
_lib.map_program_free.restype = None
_lib.map_status_str.argtypes = [ctypes.c_int]
_lib.map_status_str.restype = ctypes.c_char_p
_lib.map_last_error.argtypes = [_P]
_lib.map_last_error.restype = ctypes.c_char_p
_lib.map_chunk_count.argtypes = [_P, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint32)]
_lib.map_chunk_count.restype = ctypes.c_int
_lib.map_generate_bucketed.argtypes = [_P, ctypes.POINTER(_Exec), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                      ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]
_lib.map_generate_bucketed.restype = ctypes.c_int
_lib.map_sort_detect.argtypes = [_P, ctypes.POINTER(_Exec), ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint64,
                                 ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
_lib.map_sort_detect.restype = ctypes.c_int
_lib.map_unpack_witness.argtypes = [_P, ctypes.c_uint32, ctypes.c_uint64, ctypes.POINTER(_Witness)]
_lib.map_unpack_witness.restype = ctypes.c_int
_lib.map_default_chunk.argtypes = [_P, ctypes.c_uint32]
_lib.map_default_chunk.restype = ctypes.c_uint64
_lib.map_rank_chunks.argtypes = [_P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                 ctypes.POINTER(ctypes.c_uint32), ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)]
_lib.map_rank_chunks.restype = ctypes.c_int
_lib.map_chunk_info.argtypes = [_P, ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(_ChunkDesc)]
_lib.map_chunk_info.restype = ctypes.c_int
_lib.map_list_races.argtypes = [_P, ctypes.POINTER(_Exec), ctypes.POINTER(_Witness), ctypes.c_uint64,
                               ctypes.POINTER(ctypes.c_uint64)]
_lib.map_list_races.restype = ctypes.c_int
_lib.map_array_name.argtypes = [_P, ctypes.c_uint32]
_lib.map_array_name.restype = ctypes.c_char_p
_lib.map_debug_dump.argtypes = [_P, ctypes.c_char_p, ctypes.c_size_t]
_lib.map_debug_dump.restype = ctypes.c_size_t
_lib.map_debug_jit_check.argtypes = [_P, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_size_t]
_lib.map_debug_jit_check.restype = ctypes.c_int
_lib.map_debug_jit_source.argtypes = [_P, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_char_p, ctypes.c_size_t]
_lib.map_debug_jit_source.restype = ctypes.c_size_t
_lib.mapc_test_fastdiv.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
_lib.mapc_test_fastdiv.restype = ctypes.c_uint32


class _Typing(ctypes.Structure):
    _fields_ = [("typable", ctypes.c_int32), ("kind", ctypes.c_int32), ("line", ctypes.c_uint32),
                ("col", ctypes.c_uint32), ("var", ctypes.c_char * 64)]


_lib.map_infer.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_size_t,
                           ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(_Typing), ctypes.c_char_p, ctypes.c_size_t]
_lib.map_infer.restype = ctypes.c_int

TYPE_KINDS = {0: "ok", 1: "data_dependent_index", 2: "data_dependent_control"}


class MapError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


@dataclass
class Witness:
    phase: int
    array: int
    block: int
    index: int
    tid_lo: int
    tid_hi: int
    kind_lo: int
    kind_hi: int
    array_name: str

    def as_tuple(self):
        return (self.phase, self.array, self.block, self.index, self.tid_lo, self.tid_hi, self.kind_lo, self.kind_hi)


@dataclass
class Result:
    verdict: int                  # 0 DRF, 1 racy
    n_accesses: int
    racy_segments: int
    n_chunks: int
    device_ms: float
    gpu_launches: int
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    witness: Optional[Witness] = None
    kernels: Optional[Dict[str, Dict[str, float]]] = None   # per kernel class: ms, launches, bytes

    @property
    def racy(self) -> bool:
        return self.verdict == 1


@dataclass
class Info:
    n_phases: int
    n_arrays: int
    n_instances: int
    n_groups: int
    max_accesses: int
    max_unit_accesses: int
    u32_mode: bool
    bytecode_ops: int


def _dims(d: Sequence[int]):
    d = tuple(int(x) for x in d) + (1, 1, 1)
    return (ctypes.c_uint32 * 3)(*d[:3])


class MapProgram:
    """A MAP compiled at one instantiation (map_compile)."""

    def __init__(self, src: str, grid: Sequence[int] = (1, 1, 1), block: Sequence[int] = (1, 1, 1),
                 params: Optional[Dict[str, int]] = None):
        params = params or {}
        names = list(params)
        self._keep = [n.encode() for n in names]
        inst = _Instance()
        inst.grid = _dims(grid)
        inst.block = _dims(block)
        inst.n_params = len(names)
        inst.param_names = (ctypes.c_char_p * max(1, len(names)))(*self._keep)
        inst.param_values = (ctypes.c_uint64 * max(1, len(names)))(*[int(params[n]) for n in names])
        h = _P()
        diag = ctypes.create_string_buffer(1024)
        raw = src.encode()
        st = _lib.map_compile(raw, len(raw), ctypes.byref(inst), ctypes.byref(h), diag, 1024)
        if st != 0:
            raise MapError(st, diag.value.decode(errors="replace"))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.map_program_free(h)
            self._h = None

    def chunk_info(self, chunk: int, chunk_max_accesses: int = 0) -> dict:
        d = _ChunkDesc()
        st = _lib.map_chunk_info(self._h, int(chunk_max_accesses), int(chunk), ctypes.byref(d))
        if st != 0:
            raise MapError(st, _lib.map_last_error(self._h).decode())
        return {f: getattr(d, f) for f, _ in _ChunkDesc._fields_}

    # ---- stage API (key-exchange multi-GPU mode) ------------
    def _exec(self, scratch, stream, chunk_max_accesses, flags=0):
        import torch
        dev = scratch.device.index if scratch.device.index is not None else torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        return _Exec(dev, ctypes.c_void_p(stream.cuda_stream), ctypes.c_void_p(scratch.data_ptr()),
                     scratch.numel() * scratch.element_size(), int(chunk_max_accesses), 0, 1, None, flags)

    def generate_bucketed(self, chunk: int, rank: int, world: int, keys_out, scratch, stream=None,
                          chunk_max_accesses: int = 0):
        """Rank `rank` of `world` generates its slice of chunk `chunk`; keys laid out by destination
        rank in keys_out (uint64/int64 CUDA tensor >= the chunk bound).  Returns per-destination counts."""
        ex = self._exec(scratch, stream, chunk_max_accesses)
        counts = (ctypes.c_uint64 * world)()
        st = _lib.map_generate_bucketed(self._h, ctypes.byref(ex), rank, world, chunk,
                                        ctypes.c_void_p(keys_out.data_ptr()), counts)
        if st != 0:
            raise MapError(st, _lib.map_last_error(self._h).decode())
        return [int(c) for c in counts]

    def sort_detect(self, chunk: int, keys, n: int, scratch, stream=None, chunk_max_accesses: int = 0,
                    detect: str = "auto"):
        """Sort + detect n device keys of chunk `chunk`: (packed witness or None, racy segment count)."""
        ex = self._exec(scratch, stream, chunk_max_accesses, DETECT_PATHS[detect])
        w, r = ctypes.c_uint64(), ctypes.c_uint64()
        st = _lib.map_sort_detect(self._h, ctypes.byref(ex), chunk, ctypes.c_void_p(keys.data_ptr() if n else 0),
                                  int(n), ctypes.byref(w), ctypes.byref(r))
        if st != 0:
            raise MapError(st, _lib.map_last_error(self._h).decode())
        return (None if w.value == 2**64 - 1 else w.value), r.value

    def unpack_witness(self, chunk: int, packed: int) -> Witness:
        w = _Witness()
        st = _lib.map_unpack_witness(self._h, chunk, packed, ctypes.byref(w))
        if st != 0:
            raise MapError(st, "bad packed witness")
        return Witness(w.phase, w.array, w.block, w.index, w.tid_lo, w.tid_hi, w.kind_lo, w.kind_hi,
                       w.array_name.decode())

    def list_races(self, cap: int = 1 << 20, scratch=None, stream=None, chunk_max_accesses: int = 0):
        """All racy segments (NEXT-4): (total count, canonical witnesses of the `cap` smallest, in order)."""
        import torch
        if scratch is None:
            scratch = torch.empty(self.scratch_bytes(chunk_max_accesses), dtype=torch.uint8, device="cuda")
        ex = self._exec(scratch, stream, chunk_max_accesses)
        buf = (_Witness * max(1, cap))()
        total = ctypes.c_uint64()
        st = _lib.map_list_races(self._h, ctypes.byref(ex), buf, int(cap), ctypes.byref(total))
        if st != 0:
            raise MapError(st, _lib.map_last_error(self._h).decode())
        k = min(cap, total.value)
        return total.value, [Witness(w.phase, w.array, w.block, w.index, w.tid_lo, w.tid_hi, w.kind_lo, w.kind_hi,
                                     w.array_name.decode()) for w in buf[:k]]

    def array_names(self):
        out = []
        while True:
            n = _lib.map_array_name(self._h, len(out))
            if n is None:
                return out
            out.append(n.decode())

    def dump(self) -> str:
        """Listing of the lowered bytecode (debugging)."""
        n = _lib.map_debug_dump(self._h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        _lib.map_debug_dump(self._h, buf, n + 1)
        return buf.value.decode()

    def jit_check(self, chunk_max_accesses: int = 0) -> str:
        """NVRTC-compile the specialised generate module (no GPU needed); '' on success, else the log."""
        buf = ctypes.create_string_buffer(4096)
        r = _lib.map_debug_jit_check(self._h, int(chunk_max_accesses), buf, 4096)
        return "" if r == 0 else (buf.value.decode(errors="replace") or f"status {r}")

    def jit_source(self, chunk: int = 0, mode: int = 1, chunk_max_accesses: int = 0) -> str:
        """The specialised generate source of one chunk (mode 0 keys, 1 direct, 2 filter; debugging)."""
        old = os.environ.get("MAPC_DEBUG_JIT_MODE")
        os.environ["MAPC_DEBUG_JIT_MODE"] = str(int(mode))
        try:
            n = _lib.map_debug_jit_source(self._h, int(chunk_max_accesses), int(chunk), None, 0)
            buf = ctypes.create_string_buffer(n + 1)
            _lib.map_debug_jit_source(self._h, int(chunk_max_accesses), int(chunk), buf, n + 1)
        finally:
            if old is None:
                del os.environ["MAPC_DEBUG_JIT_MODE"]
            else:
                os.environ["MAPC_DEBUG_JIT_MODE"] = old
        return buf.value.decode()

    @property
    def info(self) -> Info:
        i = _Info()
        _lib.map_info_get(self._h, ctypes.byref(i))
        return Info(i.n_phases, i.n_arrays, i.n_instances, i.n_groups, i.max_accesses, i.max_unit_accesses,
                    bool(i.u32_mode), i.bytecode_ops)

    def scratch_bytes(self, chunk_max_accesses: int = 0) -> int:
        n = _lib.map_scratch_bytes(self._h, int(chunk_max_accesses))
        if n == 0:
            raise MapError(9, _lib.map_last_error(self._h).decode())
        return n

    def default_chunk(self, world: int = 1) -> int:
        """map_default_chunk: the chunk capacity a `world`-rank job uses by default."""
        return int(_lib.map_default_chunk(self._h, int(world)))

    def rank_chunks(self, rank: int, world: int, chunk_max_accesses: int = 0):
        """map_rank_chunks: the chunk indices rank `rank` of `world` processes."""
        n = ctypes.c_uint32()
        st = _lib.map_rank_chunks(self._h, int(chunk_max_accesses), int(rank), int(world), None, 0, ctypes.byref(n))
        if st != 0:
            raise MapError(st, _lib.map_last_error(self._h).decode())
        buf = (ctypes.c_uint32 * max(1, n.value))()
        _lib.map_rank_chunks(self._h, int(chunk_max_accesses), int(rank), int(world), buf, n.value, ctypes.byref(n))
        return list(buf[:n.value])

    def n_chunks(self, chunk_max_accesses: int = 0) -> int:
        c = ctypes.c_uint32()
        st = _lib.map_chunk_count(self._h, int(chunk_max_accesses), ctypes.byref(c))
        if st != 0:
            raise MapError(st, _lib.map_last_error(self._h).decode())
        return c.value

    def check_races(self, scratch=None, stream=None, chunk_max_accesses: int = 0, device: Optional[int] = None,
                    rank: int = 0, world: int = 1, profile: bool = False, gen: str = "auto",
                    detect: str = "auto", overlap: bool = True) -> Result:
        """Run generate -> sort -> detect on one GPU (blocking).

        scratch: a torch uint8 CUDA tensor of >= scratch_bytes() bytes (allocated here if None);
        stream: a torch.cuda.Stream (default: the current stream);
        rank/world: process only rank `rank`'s chunks (rank_chunks; multi-GPU sharding; with
                    chunk_max_accesses 0 the plan uses default_chunk(world));
        profile: record CUDA events around every launch and return per-kernel-class timings
                 (True), or around the generate launches only ("generate": the other classes are
                 counted, not timed; MAP_EXEC_PROFILE_GENERATE), or around every fourth chunk's
                 generate ("sampled": MAP_EXEC_PROFILE_SAMPLED); kernels[k]["timed"] counts them;
        gen: generate path, "auto" | "vm" (bytecode interpreter) | "jit" (NVRTC-specialised);
        detect: "auto" | "direct" | "table" | "sort" (include/mapcheck.h MAP_DETECT_*);
        overlap: False = MAP_EXEC_SEQUENTIAL (the direct path's chunks one after another)."""
        import torch
        if not torch.cuda.is_available():
            raise MapError(6, "no CUDA device (there is no CPU fallback)")
        dev = torch.cuda.current_device() if device is None else int(device)
        if not chunk_max_accesses and world > 1:
            chunk_max_accesses = self.default_chunk(world)
        need = self.scratch_bytes(chunk_max_accesses)
        if scratch is None:
            scratch = torch.empty(need, dtype=torch.uint8, device=f"cuda:{dev}")
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        stats = _Stats() if profile else None
        ex = _Exec(dev, ctypes.c_void_p(stream.cuda_stream), ctypes.c_void_p(scratch.data_ptr()),
                   scratch.numel() * scratch.element_size(), int(chunk_max_accesses), int(rank), int(world),
                   ctypes.pointer(stats) if stats is not None else None,
                   GEN_PATHS[gen] | DETECT_PATHS[detect] | (0 if overlap else EXEC_SEQUENTIAL) |
                   (EXEC_PROFILE_GENERATE if profile in ("generate", "sampled") else 0) |
                   (EXEC_PROFILE_SAMPLED if profile == "sampled" else 0))
        r = _Result()
        st = _lib.map_check_races(self._h, ctypes.byref(ex), ctypes.byref(r))
        if st != 0:
            raise MapError(st, _lib.map_last_error(self._h).decode())
        res = Result(r.verdict, r.n_accesses, r.racy_segments, r.n_chunks, r.device_ms, r.gpu_launches,
                     r.h2d_bytes, r.d2h_bytes)
        if r.verdict:
            w = _Witness()
            if _lib.map_witness_get(self._h, ctypes.byref(w)) == 0:
                res.witness = Witness(w.phase, w.array, w.block, w.index, w.tid_lo, w.tid_hi, w.kind_lo, w.kind_hi,
                                      w.array_name.decode())
        if stats is not None:
            res.kernels = {k: {"ms": stats.ms[i], "launches": stats.launches[i], "bytes": stats.bytes[i],
                               "timed": stats.timed[i]} for i, k in enumerate(KERNEL_CLASSES)}
        return res


@dataclass
class Inference:
    """map_infer: the typing outcome of a BabyCUDA kernel and its MAP text."""
    typable: bool
    kind: str                     # "ok" | "data_dependent_index" | "data_dependent_control"
    var: str
    line: int
    col: int
    map_text: Optional[str]       # None when ill-typed and no data domain was given


def infer(src: str, data_domain: int = 0) -> Inference:
    """Type a BabyCUDA kernel (Fig. 6) and infer its MAP (include/mapcheck.h map_infer)."""
    raw = src.encode()
    ty = _Typing()
    n = ctypes.c_size_t()
    diag = ctypes.create_string_buffer(1024)
    cap = 4 * len(raw) + 4096
    while True:
        buf = ctypes.create_string_buffer(cap)
        st = _lib.map_infer(raw, len(raw), int(data_domain), buf, cap, ctypes.byref(n), ctypes.byref(ty), diag, 1024)
        if st == 0 and n.value >= cap:
            cap = n.value + 1
            continue
        break
    if st not in (0, 10):
        raise MapError(st, diag.value.decode(errors="replace"))
    return Inference(bool(ty.typable), TYPE_KINDS[ty.kind], ty.var.decode(), ty.line, ty.col,
                     buf.value.decode() if st == 0 else None)


def check(src: str, grid=(1, 1, 1), block=(1, 1, 1), params=None, chunk_max_accesses: int = 0, **kw) -> Result:
    """Compile and check a MAP in one call."""
    return MapProgram(src, grid, block, params).check_races(chunk_max_accesses=chunk_max_accesses, **kw)


def status_str(status: int) -> str:
    return _lib.map_status_str(status).decode()


_lib.map_scratch_alloc.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(ctypes.c_void_p),
                                   ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32)]
_lib.map_scratch_alloc.restype = ctypes.c_int
_lib.map_scratch_free.argtypes = [ctypes.c_void_p]
_lib.map_scratch_free.restype = ctypes.c_int
EXPORTS = EXPORTS + ("map_scratch_alloc", "map_scratch_free")


class _ScratchBlock:
    """A map_scratch_alloc block, exposed through __cuda_array_interface__ so that
    torch.as_tensor wraps it without a copy; freed when the last tensor on it dies."""

    def __init__(self, nbytes: int, device: int, compressible: bool):
        ptr, size, comp = ctypes.c_void_p(), ctypes.c_uint64(), ctypes.c_uint32()
        st = _lib.map_scratch_alloc(device, int(nbytes), 1 if compressible else 0, ctypes.byref(ptr),
                                    ctypes.byref(size), ctypes.byref(comp))
        if st != 0:
            raise MapError(st, f"map_scratch_alloc({nbytes} B): {status_str(st)}")
        self.ptr, self.size, self.compressed = int(ptr.value), int(size.value), bool(comp.value)
        self._free = _lib.map_scratch_free          # held: module globals may be gone at exit
        self.__cuda_array_interface__ = {"shape": (self.size,), "typestr": "|u1", "data": (self.ptr, False),
                                         "version": 3, "strides": None}

    def __del__(self):
        if getattr(self, "ptr", 0):
            self._free(self.ptr)
            self.ptr = 0


def alloc_scratch(nbytes: int, device: Optional[int] = None, compressible: bool = True):
    """Device scratch (a torch uint8 CUDA tensor) from map_scratch_alloc: compressible
    memory when the device grants it (the direct path's cleared tables then cost fewer
    DRAM bytes, include/mapcheck.h), else plain device memory.  `.compressed` on the
    returned tensor's `_map_block` says which."""
    import torch
    dev = torch.cuda.current_device() if device is None else int(device)
    blk = _ScratchBlock(nbytes, dev, compressible)
    t = torch.as_tensor(blk, device=f"cuda:{dev}")
    t._map_block = blk
    return t


def fastdiv_selftest(n: int, d: int) -> int:
    """Host copy of the kernels' invariant-divisor quotient (for CPU tests)."""
    return _lib.mapc_test_fastdiv(n, d)


# ---- BabyCUDA executor + Theorem-1 differential check (NEXT-2) ---------------
class _KInfo(ctypes.Structure):
    _fields_ = [("typable", ctypes.c_int32), ("n_phases", ctypes.c_uint32), ("n_arrays", ctypes.c_uint32),
                ("block_threads", ctypes.c_uint32), ("n_blocks", ctypes.c_uint64),
                ("cells_per_block", ctypes.c_uint64), ("key_bits", ctypes.c_uint32), ("max_events", ctypes.c_uint64)]


class _ExecResult(ctypes.Structure):
    _fields_ = [("verdict", ctypes.c_int32), ("typable", ctypes.c_int32), ("n_events", ctypes.c_uint64),
                ("n_alpha", ctypes.c_uint64), ("racy_segments", ctypes.c_uint64), ("uninit_reads", ctypes.c_uint64),
                ("ambiguous_reads", ctypes.c_uint64), ("device_ms", ctypes.c_float), ("gpu_launches", ctypes.c_uint32)]


class _Access(ctypes.Structure):
    _fields_ = [("phase", ctypes.c_uint32), ("array", ctypes.c_uint32), ("block", ctypes.c_uint32),
                ("index", ctypes.c_uint64), ("tid", ctypes.c_uint32), ("kind", ctypes.c_uint8)]


class _Diff(ctypes.Structure):
    _fields_ = [("equal", ctypes.c_int32), ("n_alpha", ctypes.c_uint64), ("n_lambda", ctypes.c_uint64),
                ("only_alpha", ctypes.c_uint64), ("only_lambda", ctypes.c_uint64),
                ("has_first_alpha", ctypes.c_int32), ("has_first_lambda", ctypes.c_int32),
                ("first_alpha", _Access), ("first_lambda", _Access), ("exec", _ExecResult)]


EXEC_KEEP_MEMORY = 0x200
_lib.map_kernel_compile.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(_Instance), ctypes.POINTER(_P),
                                    ctypes.c_char_p, ctypes.c_size_t]
_lib.map_kernel_compile.restype = ctypes.c_int
_lib.map_kernel_info_get.argtypes = [_P, ctypes.POINTER(_KInfo)]
_lib.map_kernel_info_get.restype = ctypes.c_int
_lib.map_kernel_scratch_bytes.argtypes = [_P, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32]
_lib.map_kernel_scratch_bytes.restype = ctypes.c_size_t
_lib.map_execute.argtypes = [_P, ctypes.POINTER(_Exec), ctypes.c_uint64, ctypes.POINTER(_ExecResult)]
_lib.map_execute.restype = ctypes.c_int
_lib.map_kernel_witness.argtypes = [_P, ctypes.POINTER(_Witness)]
_lib.map_kernel_witness.restype = ctypes.c_int
_lib.map_kernel_memory.argtypes = [_P, ctypes.POINTER(_Exec), ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint8), ctypes.c_uint64]
_lib.map_kernel_memory.restype = ctypes.c_int
_lib.map_theorem1_diff.argtypes = [_P, _P, ctypes.POINTER(_Exec), ctypes.POINTER(_Exec), ctypes.c_uint64,
                                   ctypes.c_uint64, ctypes.POINTER(_Diff)]
_lib.map_theorem1_diff.restype = ctypes.c_int
_lib.map_kernel_free.argtypes = [_P]
_lib.map_kernel_free.restype = None
_lib.map_kernel_last_error.argtypes = [_P]
_lib.map_kernel_last_error.restype = ctypes.c_char_p
_lib.map_kernel_debug_source.argtypes = [_P, ctypes.c_char_p, ctypes.c_size_t]
_lib.map_kernel_debug_source.restype = ctypes.c_size_t
_lib.map_kernel_debug_jit_check.argtypes = [_P, ctypes.c_char_p, ctypes.c_size_t]
_lib.map_kernel_debug_jit_check.restype = ctypes.c_int
EXPORTS = EXPORTS + ("map_kernel_compile", "map_kernel_info_get", "map_kernel_scratch_bytes", "map_execute",
                     "map_kernel_witness", "map_kernel_memory", "map_theorem1_diff", "map_kernel_free")


@dataclass
class ExecResult:
    verdict: int
    typable: bool
    n_events: int
    n_alpha: int
    racy_segments: int
    uninit_reads: int
    ambiguous_reads: int
    device_ms: float
    gpu_launches: int
    witness: Optional[Witness] = None


@dataclass
class Diff:
    equal: bool
    n_alpha: int
    n_lambda: int
    only_alpha: int
    only_lambda: int
    first_alpha: Optional[tuple]      # (phase, array, block, index, tid, kind)
    first_lambda: Optional[tuple]
    exec: ExecResult


def _acc(a):
    return (a.phase, a.array, a.block, a.index, a.tid, a.kind)


class Kernel:
    """A BabyCUDA kernel planned at one instantiation (map_kernel_compile)."""

    def __init__(self, src: str, grid: Sequence[int] = (1, 1, 1), block: Sequence[int] = (1, 1, 1),
                 params: Optional[Dict[str, int]] = None):
        params = params or {}
        names = list(params)
        self._keep = [n.encode() for n in names]
        inst = _Instance()
        inst.grid = _dims(grid)
        inst.block = _dims(block)
        inst.n_params = len(names)
        inst.param_names = (ctypes.c_char_p * max(1, len(names)))(*self._keep)
        inst.param_values = (ctypes.c_uint64 * max(1, len(names)))(*[int(params[n]) for n in names])
        h = _P()
        diag = ctypes.create_string_buffer(1024)
        raw = src.encode()
        st = _lib.map_kernel_compile(raw, len(raw), ctypes.byref(inst), ctypes.byref(h), diag, 1024)
        if st != 0:
            raise MapError(st, diag.value.decode(errors="replace"))
        self._h = h
        self.src, self.grid, self.block, self.params = src, tuple(grid), tuple(block), dict(params)
        self._scratch = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.map_kernel_free(h)
            self._h = None

    @property
    def info(self) -> dict:
        i = _KInfo()
        _lib.map_kernel_info_get(self._h, ctypes.byref(i))
        return {f: getattr(i, f) for f, _ in _KInfo._fields_}

    def source(self) -> str:
        n = _lib.map_kernel_debug_source(self._h, None, 0)
        buf = ctypes.create_string_buffer(n + 1)
        _lib.map_kernel_debug_source(self._h, buf, n + 1)
        return buf.value.decode()

    def jit_check(self) -> str:
        """NVRTC-compile the executor (no GPU needed): '' on success, else the log."""
        buf = ctypes.create_string_buffer(8192)
        r = _lib.map_kernel_debug_jit_check(self._h, buf, 8192)
        return "" if r == 0 else (buf.value.decode(errors="replace") or f"status {r}")

    def _ex(self, scratch, stream, flags):
        import torch
        dev = scratch.device.index if scratch.device.index is not None else torch.cuda.current_device()
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        return _Exec(dev, ctypes.c_void_p(stream.cuda_stream), ctypes.c_void_p(scratch.data_ptr()),
                     scratch.numel() * scratch.element_size(), 0, 0, 1, None, flags)

    def _err(self, st):
        raise MapError(st, _lib.map_kernel_last_error(self._h).decode())

    def _result(self, r) -> ExecResult:
        out = ExecResult(r.verdict, bool(r.typable), r.n_events, r.n_alpha, r.racy_segments, r.uninit_reads,
                         r.ambiguous_reads, r.device_ms, r.gpu_launches)
        if r.verdict:
            w = _Witness()
            if _lib.map_kernel_witness(self._h, ctypes.byref(w)) == 0:
                out.witness = Witness(w.phase, w.array, w.block, w.index, w.tid_lo, w.tid_hi, w.kind_lo, w.kind_hi,
                                      w.array_name.decode())
        return out

    def execute(self, max_events: int = 0, keep_memory: bool = False, scratch=None, stream=None) -> ExecResult:
        """Run the kernel with data on the GPU and race-check the executed accesses (map_execute)."""
        import torch
        if not torch.cuda.is_available():
            raise MapError(6, "no CUDA device (there is no CPU fallback)")
        cap = int(max_events) or max(1, self.info["max_events"]) or 1 << 20
        flags = EXEC_KEEP_MEMORY if keep_memory else 0
        need = _lib.map_kernel_scratch_bytes(self._h, cap, 0, flags)
        if scratch is None:
            scratch = torch.empty(need, dtype=torch.uint8, device="cuda")
        self._scratch, self._flags = scratch, flags
        r = _ExecResult()
        st = _lib.map_execute(self._h, ctypes.byref(self._ex(scratch, stream, flags)), cap, ctypes.byref(r))
        if st == 9 and not max_events and r.n_events > cap:        # an ill-typed kernel ran longer: retry once
            return self.execute(max_events=r.n_events, keep_memory=keep_memory, stream=stream)
        if st != 0:
            self._err(st)
        return self._result(r)

    def memory(self, block: int, array: int, n: int):
        """Final contents of array `array` of block `block` after execute(keep_memory=True):
        a list of n values, None where never written."""
        vals = (ctypes.c_uint64 * max(1, n))()
        defs = (ctypes.c_uint8 * max(1, n))()
        st = _lib.map_kernel_memory(self._h, ctypes.byref(self._ex(self._scratch, None, self._flags)), block, array,
                                    vals, defs, n)
        if st != 0:
            self._err(st)
        return [vals[i] if defs[i] else None for i in range(n)]

    def theorem1_diff(self, lambda_prog: "MapProgram", max_events: int = 0, lambda_cap: int = 0) -> Diff:
        """Execute and compare the executed access values with the MAP program's Lambda (map_theorem1_diff)."""
        import torch
        cap = int(max_events) or max(1, self.info["max_events"]) or 1 << 20
        lcap = int(lambda_cap) or max(1, lambda_prog.info.max_accesses)
        scratch = torch.empty(_lib.map_kernel_scratch_bytes(self._h, cap, lcap, 0), dtype=torch.uint8, device="cuda")
        lscratch = torch.empty(lambda_prog.scratch_bytes(), dtype=torch.uint8, device="cuda")
        d = _Diff()
        st = _lib.map_theorem1_diff(self._h, lambda_prog._h, ctypes.byref(self._ex(scratch, None, 0)),
                                    ctypes.byref(lambda_prog._exec(lscratch, None, 0)), cap, lcap, ctypes.byref(d))
        if st == 9 and not max_events and d.exec.n_events > cap:
            return self.theorem1_diff(lambda_prog, max_events=d.exec.n_events, lambda_cap=lambda_cap)
        if st != 0:
            self._err(st)
        return Diff(bool(d.equal), d.n_alpha, d.n_lambda, d.only_alpha, d.only_lambda,
                    _acc(d.first_alpha) if d.has_first_alpha else None,
                    _acc(d.first_lambda) if d.has_first_lambda else None, self._result(d.exec))


def check_kernel(src: str, grid=(1, 1, 1), block=(1, 1, 1), params=None, data_domain: int = 0) -> dict:
    """One call: type the BabyCUDA kernel, race-check its MAP on the GPU, and label
    the verdict -- a race on a typable kernel is a TRUE alarm (Theorem 1,
    PAPER.md:903-918); on an ill-typed one (checked through the data-abstracted MAP
    when data_domain > 0) it may be false."""
    inf = infer(src, data_domain)
    out = {"typable": inf.typable, "type_error": None if inf.typable else (inf.kind, inf.var, inf.line, inf.col),
           "map": inf.map_text, "result": None, "true_alarm": None}
    if inf.map_text is not None:
        r = MapProgram(inf.map_text, grid, block, params).check_races()
        out["result"] = r
        out["true_alarm"] = bool(r.verdict and inf.typable)
    return out

_lib.map_kernel_extent.argtypes = [_P, ctypes.c_uint32]
_lib.map_kernel_extent.restype = ctypes.c_uint64
EXPORTS = EXPORTS + ("map_kernel_extent",)
Kernel.extents = property(lambda self: [int(_lib.map_kernel_extent(self._h, a)) for a in range(self.info["n_arrays"])])
