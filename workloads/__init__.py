"""Seeded, synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no access enumeration, no race
test, no key layout).  It only produces MAP *texts* plus the instantiation
(grid, block, parameter values) that both independent implementations consume:

* ``config(name, **sizes)`` -- the five BASELINE.json workload families as
  concrete MAP texts in the grammar of DESIGN.md §3, with their
  racy variants, optionally scaled down so the oracle finishes in seconds.
* ``workloads.fuzz`` -- a seeded random MAP generator (text + a plain data AST)
  in the spirit of SPEC.md:474-482 (``generate_typable_kernel``).

The MAPs follow the paper's protocol syntax (Fig. 2): accesses
``rd[n]``/``wr[n]``, ``;``, ``if``, ``forU``, plus the synchronized fragment
``sync``/``forS`` (read as in DESIGN.md "Readings" R7/R8).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, Tuple

__all__ = ["Instance", "config", "CONFIG_NAMES", "FULL"]


@dataclass
class Instance:
    """A MAP text instantiated at fixed grid/block dims and parameter values."""

    name: str
    src: str
    grid: Tuple[int, int, int] = (1, 1, 1)
    block: Tuple[int, int, int] = (1, 1, 1)
    params: Dict[str, int] = field(default_factory=dict)

    @property
    def n_threads(self) -> int:
        return self.block[0] * self.block[1] * self.block[2]

    @property
    def n_blocks(self) -> int:
        return self.grid[0] * self.grid[1] * self.grid[2]


# ---------------------------------------------------------------------------
# Config 1: the paper's worked examples.
#   1a  Fig. 3 right column, PAPER.md:279-282  "forU x in 0..M { rd[x]; wr[x] }"
#   1b  Fig. 4 right column, PAPER.md:366-369  "if (tid=0) { wr[0] } else { skip }"
# ---------------------------------------------------------------------------
_SRC_1A = "params M; forU x in 0..M { rd[x]; wr[x] }"
_SRC_1B = "if (tid = 0) { wr[0] } else { skip }"

# ---------------------------------------------------------------------------
# Config 2: shared-memory tree reduction, blockDim = 2H, L = log2(2H) phases.
#   2a DRF; 2b loop sync removed (forS -> forU); 2c first sync removed.
# ---------------------------------------------------------------------------
_SRC_2A = """params H, L; shared s;
wr s[tid]; sync;
forS k in 0..L {
  if (tid < (H >> k)) { rd s[tid]; rd s[tid + (H >> k)]; wr s[tid] } else { skip };
  sync
}"""
_SRC_2B = """params H, L; shared s;
wr s[tid]; sync;
forU k in 0..L {
  if (tid < (H >> k)) { rd s[tid]; rd s[tid + (H >> k)]; wr s[tid] } else { skip }
}"""
_SRC_2C = """params H, L; shared s;
wr s[tid];
forS k in 0..L {
  if (tid < (H >> k)) { rd s[tid]; rd s[tid + (H >> k)]; wr s[tid] } else { skip };
  sync
}"""

# ---------------------------------------------------------------------------
# Config 3: TSxTS tiled transpose, blockDim = TS x RW, each thread TS/RW rows.
#   3a with __syncthreads (DRF); 3b without (racy).
# ---------------------------------------------------------------------------
_SRC_3A = """params TS, RW; shared tile;
forU j in 0..TS step RW { wr tile[(tid / TS + j) * TS + tid % TS] };
sync;
forU j in 0..TS step RW { rd tile[(tid % TS) * TS + tid / TS + j] }"""
_SRC_3B = """params TS, RW; shared tile;
forU j in 0..TS step RW { wr tile[(tid / TS + j) * TS + tid % TS] };
forU j in 0..TS step RW { rd tile[(tid % TS) * TS + tid / TS + j] }"""

# ---------------------------------------------------------------------------
# Config 4: scans over N elements with blockDim = BS, D = log2(N) levels.
#   4a Hillis-Steele double buffered (DRF); 4b in place (racy);
#   4c Blelloch (DRF); 4d Blelloch without down-sweep syncs (racy).
# ---------------------------------------------------------------------------
_SRC_4A = """params N, D, BS; shared temp;
forS d in 0..D {
  forU k in 0..N / BS {
    if (k * BS + tid >= (1 << d)) {
      rd temp[(d % 2) * N + k * BS + tid - (1 << d)];
      rd temp[(d % 2) * N + k * BS + tid];
      wr temp[((d + 1) % 2) * N + k * BS + tid]
    } else {
      rd temp[(d % 2) * N + k * BS + tid];
      wr temp[((d + 1) % 2) * N + k * BS + tid]
    }
  };
  sync
}"""
_SRC_4B = """params N, D, BS; shared temp;
forS d in 0..D {
  forU k in 0..N / BS {
    if (k * BS + tid >= (1 << d)) {
      rd temp[k * BS + tid - (1 << d)];
      rd temp[k * BS + tid];
      wr temp[k * BS + tid]
    } else { skip }
  };
  sync
}"""
_BLELLOCH_HEAD = """params N, D, BS; shared temp;
forU k in 0..N / BS { wr temp[k * BS + tid] };
sync;
forS l in 0..D {
  forU k in 0..((N >> (l + 1)) + BS - 1) / BS {
    if (k * BS + tid < (N >> (l + 1))) {
      rd temp[(1 << l) * (2 * (k * BS + tid) + 1) - 1];
      rd temp[(1 << l) * (2 * (k * BS + tid) + 2) - 1];
      wr temp[(1 << l) * (2 * (k * BS + tid) + 2) - 1]
    } else { skip }
  };
  sync
};
if (tid = 0) { wr temp[N - 1] } else { skip };
sync;
"""
_BLELLOCH_DOWN_BODY = """forU k in 0..((1 << l) + BS - 1) / BS {
    if (k * BS + tid < (1 << l)) {
      rd temp[(N >> (l + 1)) * (2 * (k * BS + tid) + 1) - 1];
      rd temp[(N >> (l + 1)) * (2 * (k * BS + tid) + 2) - 1];
      wr temp[(N >> (l + 1)) * (2 * (k * BS + tid) + 1) - 1];
      rd temp[(N >> (l + 1)) * (2 * (k * BS + tid) + 2) - 1];
      wr temp[(N >> (l + 1)) * (2 * (k * BS + tid) + 2) - 1]
    } else { skip }
  }"""
_SRC_4C = _BLELLOCH_HEAD + "forS l in 0..D {\n  " + _BLELLOCH_DOWN_BODY + ";\n  sync\n}"
_SRC_4D = _BLELLOCH_HEAD + "forU l in 0..D {\n  " + _BLELLOCH_DOWN_BODY + "\n}"

# ---------------------------------------------------------------------------
# Config 5: synthetic 3-deep loop stencil; thread tid owns rows [tid*R, tid*R+R)
# of an H x C grid (H = blockDim * R), periodic in rows, T time steps.
#   5a ping-pong between two halves (DRF); 5b in place (racy).
# ---------------------------------------------------------------------------
_SRC_5A = """params T, R, C, H; shared A;
forS t in 0..T {
  forU r in 0..R {
    forU c in 0..C {
      rd A[(t % 2) * H * C + ((tid * R + r + H - 1) % H) * C + c];
      rd A[(t % 2) * H * C + (tid * R + r) * C + c];
      rd A[(t % 2) * H * C + ((tid * R + r + 1) % H) * C + c];
      wr A[((t + 1) % 2) * H * C + (tid * R + r) * C + c]
    }
  };
  sync
}"""
_SRC_5B = """params T, R, C, H; shared A;
forS t in 0..T {
  forU r in 0..R {
    forU c in 0..C {
      rd A[((tid * R + r + H - 1) % H) * C + c];
      rd A[(tid * R + r) * C + c];
      rd A[((tid * R + r + 1) % H) * C + c];
      wr A[(tid * R + r) * C + c]
    }
  };
  sync
}"""

# Full BASELINE.json sizes.
FULL = {
    "1a": dict(block=8, M=8),
    "1b": dict(block=8),
    "2a": dict(block=1024), "2b": dict(block=1024), "2c": dict(block=1024),
    "3a": dict(ts=32, rw=8, grid=65536), "3b": dict(ts=32, rw=8, grid=65536),
    "4a": dict(n=1 << 20, bs=1024), "4b": dict(n=1 << 20, bs=1024),
    "4c": dict(n=1 << 20, bs=1024), "4d": dict(n=1 << 20, bs=1024),
    "5a": dict(block=1024, T=16, R=256, C=1024),
    "5b": dict(block=1024, T=16, R=256, C=1024),
}
CONFIG_NAMES = tuple(FULL)


def _log2(x: int) -> int:
    if x <= 0 or x & (x - 1):
        raise ValueError(f"{x} is not a power of two")
    return x.bit_length() - 1


def config(name: str, **sizes) -> Instance:
    """Instance of config ``name`` at the given sizes (defaults: full size)."""
    s = dict(FULL[name])
    s.update(sizes)
    fam = name[0]
    if name == "1a":
        return Instance(name, _SRC_1A, block=(s["block"], 1, 1), params={"M": s["M"]})
    if name == "1b":
        return Instance(name, _SRC_1B, block=(s["block"], 1, 1))
    if fam == "2":
        b = s["block"]
        src = {"2a": _SRC_2A, "2b": _SRC_2B, "2c": _SRC_2C}[name]
        return Instance(name, src, block=(b, 1, 1), params={"H": b // 2, "L": _log2(b)})
    if fam == "3":
        ts, rw = s["ts"], s["rw"]
        src = _SRC_3A if name == "3a" else _SRC_3B
        return Instance(name, src, grid=(s["grid"], 1, 1), block=(ts, rw, 1),
                        params={"TS": ts, "RW": rw})
    if fam == "4":
        n, bs = s["n"], s["bs"]
        src = {"4a": _SRC_4A, "4b": _SRC_4B, "4c": _SRC_4C, "4d": _SRC_4D}[name]
        return Instance(name, src, block=(bs, 1, 1), params={"N": n, "D": _log2(n), "BS": bs})
    if fam == "5":
        b, R, C, T = s["block"], s["R"], s["C"], s["T"]
        src = _SRC_5A if name == "5a" else _SRC_5B
        return Instance(name, src, block=(b, 1, 1),
                        params={"T": T, "R": R, "C": C, "H": b * R})
    raise KeyError(name)
