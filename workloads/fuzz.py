"""Seeded random MAP generator (test inputs only; no method arithmetic here).

Produces a plain-data AST (tuples) and its MAP text.  The same AST is evaluated
by the pure-Python brute force (tests/brute.py) while the text goes to the C++
oracle and to the CUDA path, so a parser bug on either side shows up as a
disagreement.  Shape limits follow SURVEY.md §4 item 3: blockDim <= 16, trip
counts <= 4, <= 3 phases, <= 2 arrays, <= 2 blocks.  In the spirit of
SPEC.md:474-482 (``generate_typable_kernel``): MAPs are data-independent by
construction (indices and guards use only tid, bid, loop variables, params and
literals).

AST node shapes
  num : ("nat", v) | ("var", name) | ("tid",) | ("bid",)
        | ("bin", op, a, b)   op in + - * / % << >> min max
  cond: ("true",) | ("false",) | ("rel", op, a, b)   op in = != < <= > >=
        | ("and", l, r) | ("or", l, r)
  stmt: ("skip",) | ("sync",) | ("acc", kind, array, idx)   kind in rd wr
        | ("seq", [stmt...]) | ("if", cond, then, else)
        | ("forU"|"forS", var, lo, hi, step, body)
  program: {"params": [names], "arrays": [names], "body": stmt}
"""
from __future__ import annotations

import random
from typing import List

from . import Instance

_ARITH = ["+", "+", "-", "*", "/", "%", "<<", ">>", "min", "max"]
_RELS = ["=", "!=", "<", "<=", ">", ">="]


class _Gen:
    def __init__(self, seed: int):
        self.r = random.Random(seed)
        self.n_loopvars = 0
        self.syncs_left = 2

    # -- expressions --------------------------------------------------------
    def leaf(self, scope: List[str], uniform: bool):
        r = self.r
        choices = ["nat", "nat"]
        if not uniform:
            choices += ["tid", "tid", "bid"]
        if scope:
            choices += ["var", "var"]
        c = r.choice(choices)
        if c == "nat":
            return ("nat", r.randint(0, 5))
        if c == "var":
            return ("var", r.choice(scope))
        return (c,)

    def num(self, scope, depth, uniform=False):
        r = self.r
        if depth <= 0 or r.random() < 0.35:
            return self.leaf(scope, uniform)
        op = r.choice(_ARITH)
        a = self.num(scope, depth - 1, uniform)
        if op in ("/", "%"):
            b = ("nat", r.randint(1, 4))           # never divide by zero
        elif op in ("<<", ">>"):
            b = ("nat", r.randint(0, 2))
        elif op == "*":
            b = ("nat", r.randint(0, 3)) if r.random() < 0.6 else self.num(scope, depth - 1, uniform)
        else:
            b = self.num(scope, depth - 1, uniform)
        return ("bin", op, a, b)

    def index(self, scope):
        # fold into a small range so distinct threads collide often
        e = self.num(scope, 2)
        return ("bin", "%", e, ("nat", self.r.randint(2, 9)))

    def cond(self, scope, depth=1):
        r = self.r
        x = r.random()
        if depth > 0 and x < 0.2:
            return (r.choice(["and", "or"]), self.cond(scope, depth - 1), self.cond(scope, depth - 1))
        if x < 0.25:
            return (r.choice(["true", "false"]),)
        return ("rel", r.choice(_RELS), self.num(scope, 1), self.num(scope, 1))

    # -- statements ---------------------------------------------------------
    def fresh(self):
        self.n_loopvars += 1
        return f"x{self.n_loopvars}"

    def bounds(self, scope, uniform):
        r = self.r
        lo = ("nat", r.randint(0, 2)) if r.random() < 0.7 else self.leaf(scope, uniform)
        span = ("nat", r.randint(0, 4)) if r.random() < 0.6 else \
            ("bin", "%", self.num(scope, 1, uniform), ("nat", r.randint(1, 5)))
        hi = ("bin", "+", lo, span)
        step = ("nat", r.choice([1, 1, 1, 2]))
        return lo, hi, step

    def u(self, scope, arrays, depth):
        r = self.r
        x = r.random()
        if depth <= 0 or x < 0.35:
            if r.random() < 0.1:
                return ("skip",)
            return ("acc", r.choice(["rd", "wr"]), r.choice(arrays), self.index(scope))
        if x < 0.55:
            return ("seq", [self.u(scope, arrays, depth - 1) for _ in range(r.randint(2, 3))])
        if x < 0.75:
            els = self.u(scope, arrays, depth - 1) if r.random() < 0.7 else ("skip",)
            return ("if", self.cond(scope), self.u(scope, arrays, depth - 1), els)
        v = self.fresh()
        lo, hi, step = self.bounds(scope, uniform=False)
        return ("forU", v, lo, hi, step, self.u(scope + [v], arrays, depth - 1))

    def p(self, scope, arrays, depth, allow_fors=True):
        r = self.r
        items = []
        for _ in range(r.randint(1, 3)):
            x = r.random()
            if x < 0.55 or depth <= 0:
                items.append(self.u(scope, arrays, 2))
            elif x < 0.8 and self.syncs_left > 0:
                self.syncs_left -= 1
                items.append(("sync",))
            elif allow_fors:
                v = self.fresh()
                lo = ("nat", r.randint(0, 1))
                hi = ("bin", "+", lo, ("nat", r.randint(0, 2)) if r.random() < 0.7
                      else self.leaf([s for s in scope if s.startswith("P")], True))
                body = self.p(scope + [v], arrays, depth - 1, allow_fors=False)
                body = ("seq", [body, ("sync",)]) if r.random() < 0.8 else body
                items.append(("forS", v, lo, hi, ("nat", 1), body))
        if not items:
            items.append(self.u(scope, arrays, 2))
        return items[0] if len(items) == 1 else ("seq", items)


def random_program(seed: int) -> dict:
    g = _Gen(seed)
    r = g.r
    params = [f"P{i}" for i in range(r.randint(0, 2))]
    n_arr = r.randint(1, 2)
    arrays = ["A", "B"][:n_arr]
    body = g.p(list(params), arrays, depth=2)
    return {"params": params, "arrays": arrays, "body": body}


def random_instance(seed: int, big_block: bool = False) -> tuple[Instance, dict]:
    """(instance, ast) for fuzz seed ``seed``; ``big_block`` draws blockDim from
    1025..2048 (as (1024, 2, 1)-shaped or flat dims) instead of <= 16."""
    prog = random_program(seed)
    r = random.Random(seed ^ 0x5EED)
    if big_block:
        n = r.randint(1025, 2048)
        block = (1024, 2, 1) if n == 2048 else (n, 1, 1)
    else:
        block = (r.choice([1, 2, 3, 4, 5, 8, 16]), 1, 1)
    grid = (r.choice([1, 1, 2]), 1, 1)
    params = {p: r.randint(0, 4) for p in prog["params"]}
    return Instance(f"fuzz{seed}", to_text(prog), grid=grid, block=block, params=params), prog


# -- printing ---------------------------------------------------------------
def num_text(e) -> str:
    k = e[0]
    if k == "nat":
        return str(e[1])
    if k == "var":
        return e[1]
    if k in ("tid", "bid"):
        return k
    _, op, a, b = e
    if op in ("min", "max"):
        return f"{op}({num_text(a)}, {num_text(b)})"
    return f"({num_text(a)} {op} {num_text(b)})"


def cond_text(c) -> str:
    k = c[0]
    if k in ("true", "false"):
        return k
    if k == "rel":
        return f"{num_text(c[2])} {c[1]} {num_text(c[3])}"
    return f"({cond_text(c[1])} {k} {cond_text(c[2])})"


def stmt_text(s, multi_array: bool) -> str:
    k = s[0]
    if k in ("skip", "sync"):
        return k
    if k == "acc":
        arr = f" {s[2]}" if multi_array else ""
        return f"{s[1]}{arr}[{num_text(s[3])}]"
    if k == "seq":
        return "; ".join(stmt_text(x, multi_array) for x in s[1])
    if k == "if":
        return (f"if ({cond_text(s[1])}) {{ {stmt_text(s[2], multi_array)} }} "
                f"else {{ {stmt_text(s[3], multi_array)} }}")
    _, v, lo, hi, step, body = s
    st = "" if step == ("nat", 1) else f" step {num_text(step)}"
    return f"{k} {v} in {num_text(lo)}..{num_text(hi)}{st} {{ {stmt_text(body, multi_array)} }}"


def to_text(prog: dict) -> str:
    parts = []
    if prog["params"]:
        parts.append("params " + ", ".join(prog["params"]) + ";")
    multi = len(prog["arrays"]) > 1
    if multi:
        parts.append("shared " + ", ".join(prog["arrays"]) + ";")
    parts.append(stmt_text(prog["body"], multi))
    return "\n".join(parts)


def random_rows_instance(seed: int) -> Instance:
    """A random two-loop MAP over rows r (second-innermost) and columns c
    (innermost), sized so that the JIT's row-jam applies (blockDim * R * C a
    multiple of 1024, C a multiple of 4 dividing or divisible by 512): sites read
    or write row (tid * R + r + a) mod H (or a row shared by every thread, or a
    row stride 2) at column c + b, some under a guard on r, c or tid.  Test input
    only."""
    r = random.Random(10_000 + seed)
    nt = r.choice([8, 16, 32, 64])
    R = r.choice([2, 4, 8])
    C = r.choice([4, 8, 16, 64, 512, 1024])
    while nt * R * C < 1024:
        C *= 2
    H = nt * R
    sites = []
    # a stencil-like family of rows (consecutive offsets: rows r + a, r + a + 1, ...
    # are touched again by the next row) plus a few unrelated sites
    fam = r.choice(["tid", "tid", "shared", "stride2"])
    a0 = r.choice([0, H - 1, 1])
    n_fam = r.randint(2, 4)
    fam_arr, fam_half, fam_b = r.choice(["A", "A", "B"]), r.choice(["", f"{2 * H + 2} * C + "]), r.choice([0, 0, 1])
    plan = [(a0 + i, fam, True) for i in range(n_fam)] + \
        [(r.choice([0, 1, 2, H - 1]), r.choice(["tid", "shared", "stride2"]), False) for _ in range(r.randint(0, 2))]
    r.shuffle(plan)
    for a, f, in_fam in plan:
        kind = r.choice(["rd", "rd", "wr"])
        arr = fam_arr if in_fam else r.choice(["A", "A", "A", "B"])
        b = fam_b if in_fam else r.choice([0, 0, 0, 1, 2, 4])
        row = {"tid": f"((tid * R + r + {a}) % H)", "shared": f"(r + {a % 3})",
               "stride2": f"(2 * (tid * R + r) + {a % 2})"}[f]
        half = fam_half if in_fam else r.choice(["", "", f"{2 * H + 2} * C + "])
        acc = f"{kind} {arr}[{half}{row} * C + c + {b}]"
        g = r.random()
        if g < 0.2:
            acc = f"if (r % 2 = {r.randint(0, 1)}) {{ {acc} }} else {{ skip }}"
        elif g < 0.3:
            acc = f"if (tid < {r.randint(1, nt)}) {{ {acc} }} else {{ skip }}"
        elif g < 0.35:
            acc = f"if (c >= {r.randint(0, C)}) {{ {acc} }} else {{ skip }}"
        sites.append(acc)
    src = "params R, C, H; shared A, B;\nforU r in 0..R { forU c in 0..C { " + "; ".join(sites) + " } }"
    if r.random() < 0.3:
        src += ";\nsync;\nforU r in 0..R { forU c in 0..C { " + "; ".join(reversed(sites)) + " } }"
    return Instance(f"rows{seed}", src, grid=(r.choice([1, 2]), 1, 1), block=(nt, 1, 1),
                    params={"R": R, "C": C, "H": H})


def random_strided_instance(seed: int) -> Instance:
    """A random MAP whose sites index with a power-of-two stride (index = s * (k * nt
    + tid + a) + b, same or different residues b, per-phase strides, guards): the
    shapes for which the direct table is stride-compressed.  Test input only."""
    r = random.Random(20_000 + seed)
    nt = r.choice([8, 16, 32, 64])
    N = r.choice([4, 16, 64])
    phases = []
    for _ in range(r.randint(1, 3)):
        s = r.choice([2, 4, 8, 16])
        base = r.randrange(s)
        sites = []
        for _ in range(r.randint(1, 4)):
            kind = r.choice(["rd", "rd", "wr"])
            arr = r.choice(["A", "A", "B"])
            a = r.choice([0, 0, 1, nt - 1])
            b = base if r.random() < 0.8 else r.randrange(s)
            t = r.choice(["tid", "tid", "(tid / 2)", "((tid + 1) % " + str(nt) + ")"])
            acc = f"{kind} {arr}[{s} * (k * {nt} + {t} + {a}) + {b}]"
            if r.random() < 0.2:
                acc = f"if (k < {r.randint(1, N)}) {{ {acc} }} else {{ skip }}"
            sites.append(acc)
        phases.append("forU k in 0..N { " + "; ".join(sites) + " }")
    src = "params N; shared A, B;\n" + ";\nsync;\n".join(phases)
    return Instance(f"strided{seed}", src, grid=(r.choice([1, 2]), 1, 1), block=(nt, 1, 1), params={"N": N})
