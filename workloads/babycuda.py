"""Seeded, synthetic BabyCUDA kernels (test and bench inputs; no method arithmetic).

BabyCUDA (Fig. 5) carries data: ``A[n] := m`` writes the value
of m, ``let y = A[n] in b`` reads A[n] into y for the rest of the block.  The
texts follow the grammar of DESIGN.md §3b and feed both the oracle
(oracle/babycuda.py) and the product (map_infer / map_execute).

* ``PAPER`` -- the paper's worked kernels: Fig. 3 (racy, PAPER.md:279-282 /
  displayed derivation :836-856), Fig. 4 (DRF, :366-369 / :858-876) and the
  ill-typed kernel of Eq. 1 (:887-891).
* ``kernel(name, **sizes)`` -- the BASELINE.json workload families written as
  data-carrying kernels (tree reduction, tiled transpose, Hillis-Steele scan,
  Blelloch scan, 3-point stencil); each one's inferred MAP has the access
  structure of the matching ``workloads.config`` MAP.
* ``random_kernel(seed, ill_typed=False)`` -- random typable kernels (indices,
  conditions and loop bounds over tid, bid, params and loop variables only;
  read values flow into payloads), or ill-typed ones (one read value reaches an
  index or a condition) -- the Theorem-1 differential corpus.
"""
from __future__ import annotations

import random
from typing import Dict, Tuple

from . import Instance

PAPER = {
    # Fig. 3 middle column: for x in 0..M { y = A[x]; A[x] = y + 1 }
    "fig3_racy": "params M; for x in 0..M { let y = A[x] in A[x] := y + 1 }",
    # Fig. 4 middle column: if (tid = 0) { A[0] := tid } else { skip }
    "fig4_drf": "if (tid = 0) { A[0] := tid } else { skip }",
    # Eq. 1: A[tid] := tid; let x = A[tid] in A[x] := 9  (ill-typed: x indexes A)
    "eq1_ill_typed": "A[tid] := tid; let x = A[tid] in A[x] := 9",
}

_REDUCE = """params H, L; shared s[{n}];
s[tid] := tid + 1; sync;
for k in 0..L {{
  if (tid < (H >> k)) {{ let a = s[tid] in let b = s[tid + (H >> k)] in s[tid] := a + b }} else {{ skip }}{sync}
}}"""

_TRANSPOSE = """params TS, RW; shared tile[{n}], out[{n}];
for j in 0..TS step RW {{ tile[(tid / TS + j) * TS + tid % TS] := bid * TS * TS + (tid / TS + j) * TS + tid % TS }};
{sync}
for j in 0..TS step RW {{ let v = tile[(tid % TS) * TS + tid / TS + j] in out[(tid / TS + j) * TS + tid % TS] := v }}"""

_HILLIS = """params N, D, BS; shared temp[{n2}];
for k in 0..N / BS {{ temp[k * BS + tid] := 1 }};
sync;
for d in 0..D {{
  for k in 0..N / BS {{
    if (k * BS + tid >= (1 << d)) {{
      let a = temp[(d % 2) * N + k * BS + tid - (1 << d)] in
      let b = temp[(d % 2) * N + k * BS + tid] in
      temp[((d + 1) % 2) * N + k * BS + tid] := a + b
    }} else {{
      let a = temp[(d % 2) * N + k * BS + tid] in temp[((d + 1) % 2) * N + k * BS + tid] := a
    }}
  }};
  sync
}}"""

_HILLIS_INPLACE = """params N, D, BS; shared temp[{n}];
for k in 0..N / BS {{ temp[k * BS + tid] := 1 }};
sync;
for d in 0..D {{
  for k in 0..N / BS {{
    if (k * BS + tid >= (1 << d)) {{
      let a = temp[k * BS + tid - (1 << d)] in let b = temp[k * BS + tid] in temp[k * BS + tid] := a + b
    }} else {{ skip }}
  }};
  sync
}}"""

_STENCIL = """params T, R, C, H; shared A[{n}];
for r in 0..R {{ for c in 0..C {{ A[(tid * R + r) * C + c] := (tid * R + r) * 3 + c }} }};
sync;
for t in 0..T {{ for r in 0..R {{ for c in 0..C {{
  let a = A[{off}((tid * R + r + H - 1) % H) * C + c] in
  let b = A[{off}(tid * R + r) * C + c] in
  let e = A[{off}((tid * R + r + 1) % H) * C + c] in
  A[{woff}(tid * R + r) * C + c] := (a + b + e) % 1000003
}} }}; sync }}"""


def kernel(name: str, **kw) -> Instance:
    """A data-carrying BabyCUDA kernel of workload family `name` at small sizes."""
    if name in ("reduce", "reduce_racy"):
        B = kw.get("block", 64)
        L = B.bit_length() - 1
        src = _REDUCE.format(n=B, sync="; sync" if name == "reduce" else "")
        return Instance(name, src, (kw.get("grid", 1), 1, 1), (B, 1, 1), {"H": B // 2, "L": L})
    if name in ("transpose", "transpose_racy"):
        ts, rw, g = kw.get("ts", 8), kw.get("rw", 4), kw.get("grid", 4)
        src = _TRANSPOSE.format(n=ts * ts, sync="sync;" if name == "transpose" else "skip;")
        return Instance(name, src, (g, 1, 1), (ts * rw, 1, 1), {"TS": ts, "RW": rw})
    if name == "hillis":
        n, bs = kw.get("n", 256), kw.get("bs", 64)
        return Instance(name, _HILLIS.format(n2=2 * n), (1, 1, 1), (bs, 1, 1),
                        {"N": n, "D": n.bit_length() - 1, "BS": bs})
    if name == "hillis_inplace":
        n, bs = kw.get("n", 256), kw.get("bs", 64)
        return Instance(name, _HILLIS_INPLACE.format(n=n), (1, 1, 1), (bs, 1, 1),
                        {"N": n, "D": n.bit_length() - 1, "BS": bs})
    if name in ("stencil", "stencil_racy"):
        B, T, R, C = kw.get("block", 16), kw.get("T", 2), kw.get("R", 2), kw.get("C", 8)
        H = B * R
        if name == "stencil":
            src = _STENCIL.format(n=2 * H * C, off="(t % 2) * H * C + ", woff="((t + 1) % 2) * H * C + ")
        else:
            src = _STENCIL.format(n=H * C, off="", woff="")
        return Instance(name, src, (1, 1, 1), (B, 1, 1), {"T": T, "R": R, "C": C, "H": H})
    raise KeyError(name)


KERNELS = ["reduce", "reduce_racy", "transpose", "transpose_racy", "hillis", "hillis_inplace", "stencil",
           "stencil_racy"]


# ------------------------------------------------------------- fuzzing ------
class _Gen:
    def __init__(self, seed: int, ill_typed: bool):
        self.r = random.Random(seed)
        self.ill = ill_typed
        self.planted = False
        self.n = 0

    def fresh(self, p):
        self.n += 1
        return f"{p}{self.n}"

    def expr(self, typed, data, depth=2):
        """An expression over `typed` names (+ `data` names when allowed)."""
        r = self.r
        names = list(typed) + list(data)
        if depth == 0 or r.random() < 0.4:
            c = r.random()
            if c < 0.35 or not names:
                return str(r.randint(0, 5))
            return r.choice(names)
        op = r.choice(["+", "+", "-", "*", "%", "/", "min", "max", ">>"])
        a = self.expr(typed, data, depth - 1)
        if op in ("%", "/"):
            return f"({a} {op} {r.randint(1, 4)})"
        if op == ">>":
            return f"({a} >> {r.randint(0, 2)})"
        b = self.expr(typed, data, depth - 1)
        return f"{op}({a}, {b})" if op in ("min", "max") else f"({a} {op} {b})"

    def index(self, typed, data):
        r = self.r
        if self.ill and data and not self.planted and r.random() < 0.5:
            self.planted = True
            return f"({r.choice(list(data))} % 6)"           # a read value reaches an index: ill-typed
        return f"({self.expr(typed, (), 2)} % 12)"

    def cond(self, typed, data):
        r = self.r
        if self.ill and data and not self.planted and r.random() < 0.3:
            self.planted = True
            return f"{r.choice(list(data))} < {r.randint(1, 4)}"
        return f"{self.expr(typed, (), 1)} {r.choice(['=', '!=', '<', '<=', '>', '>='])} {self.expr(typed, (), 1)}"

    def block(self, typed, data, arrays, depth, allow_sync):
        r = self.r
        out = []
        for _ in range(r.randint(1, 3)):
            c = r.random()
            if c < 0.3:
                out.append(f"{r.choice(arrays)}[{self.index(typed, data)}] := {self.expr(typed, data, 2)}")
            elif c < 0.5 and depth > 0:
                y = self.fresh("y")
                head = f"let {y} = {r.choice(arrays)}[{self.index(typed, data)}] in "
                out.append(head + self.block(typed, data + [y], arrays, depth - 1, allow_sync))
                break                                           # the let took the rest of the block
            elif c < 0.65 and depth > 0:
                out.append(f"if ({self.cond(typed, data)}) {{ {self.block(typed, data, arrays, depth - 1, False)} }} "
                           f"else {{ {self.block(typed, data, arrays, depth - 1, False)} }}")
            elif c < 0.8 and depth > 0:
                x = self.fresh("x")
                lo, hi = r.randint(0, 2), r.randint(0, 4)
                st = f" step {r.randint(1, 2)}" if r.random() < 0.2 else ""
                body_sync = allow_sync and r.random() < 0.3
                body = self.block(typed + [x], data, arrays, depth - 1, body_sync)
                if body_sync:
                    body += "; sync"
                out.append(f"for {x} in {lo}..{hi}{st} {{ {body} }}")
            elif c < 0.9 and allow_sync:
                out.append("sync")
            else:
                out.append("skip")
        return "; ".join(out)


def random_kernel(seed: int, ill_typed: bool = False) -> Tuple[Instance, bool]:
    """(instance, planted) -- a random kernel; `planted` tells whether an
    ill-typed use of a read value was actually placed (ill_typed requests one)."""
    g = _Gen(seed, ill_typed)
    r = g.r
    params = [f"P{i}" for i in range(r.randint(0, 2))]
    arrays = ["A", "B"][:r.randint(1, 2)]
    body = g.block(["tid", "bid"] + params, [], arrays, 3, True)
    head = (f"params {', '.join(params)}; " if params else "") + f"shared {', '.join(a + '[16]' for a in arrays)}; "
    rr = random.Random(seed ^ 0xBABE)
    block = (rr.choice([1, 2, 3, 4, 8]), 1, 1)
    grid = (rr.choice([1, 1, 2]), 1, 1)
    vals: Dict[str, int] = {p: rr.randint(0, 3) for p in params}
    return Instance(f"bfuzz{seed}", head + body, grid, block, vals), g.planted
