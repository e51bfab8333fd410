"""L0 brute force -- pins the C++ oracle (test infrastructure only).

Two independent ways to produce the access multiset, neither of which parses
MAP text:
  * ``CONFIG_LOOPS[name](...)`` -- each BASELINE.json config written directly as
    Python loops (the MAP of SURVEY.md §8d transcribed by hand), and
  * ``eval_ast(prog, ...)`` -- a direct evaluator of the fuzz generator's
    plain-data AST (workloads/fuzz.py), following the per-thread rules of
    PAPER.md:479-558 with data erased and the par union of PAPER.md:579-589.
The race test is the definition of PAPER.md:111-113 checked over ALL pairs of
accesses (no bucketing beyond equality of (phase, array, block, index)), so it
is only used on small inputs.
"""
from __future__ import annotations

import itertools
from collections import defaultdict

RD, WR = 0, 1


# --------------------------------------------------------------------------
# race definition on a list of access records (phase, array, block, index, tid, kind)
# --------------------------------------------------------------------------
def races(records):
    """(verdict, witness, n_racy_segments, n_accesses) by naive pair testing.

    witness = lexicographic min of (phase, array, block, index, t_lo, t_hi, k_lo, k_hi).
    """
    n = len(records)
    groups = defaultdict(set)      # Lambda is a set
    for (ph, ar, bl, ix, t, k) in records:
        groups[(ph, ar, bl, ix)].add((t, k))
    best = None
    racy_segments = 0
    for key, vals in groups.items():
        seg_racy = False
        for (t1, k1), (t2, k2) in itertools.combinations(sorted(vals), 2):
            if t1 == t2 or (k1 == RD and k2 == RD):
                continue
            lo, hi = ((t1, k1), (t2, k2)) if t1 < t2 else ((t2, k2), (t1, k1))
            cand = key + (lo[0], hi[0], lo[1], hi[1])
            if best is None or cand < best:
                best = cand
            seg_racy = True
        racy_segments += seg_racy
    return (1 if best is not None else 0), best, racy_segments, n


def race_list(records):
    """Every racy (phase, array, block, index) cell's minimal pair, sorted: the
    per-segment listing of SPEC.md:434-437 races_of, by naive pair testing."""
    groups = defaultdict(set)
    for (ph, ar, bl, ix, t, k) in records:
        groups[(ph, ar, bl, ix)].add((t, k))
    out = []
    for key, vals in groups.items():
        best = None
        for (t1, k1), (t2, k2) in itertools.combinations(sorted(vals), 2):
            if t1 == t2 or (k1 == RD and k2 == RD):
                continue
            lo, hi = ((t1, k1), (t2, k2)) if t1 < t2 else ((t2, k2), (t1, k1))
            cand = key + (lo[0], hi[0], lo[1], hi[1])
            if best is None or cand < best:
                best = cand
        if best is not None:
            out.append(best)
    return sorted(out)


def races_all_pairs(records):
    """Same verdict/witness by testing every pair of the whole multiset (O(N^2))."""
    best = None
    for a, b in itertools.combinations(records, 2):
        if a[:4] != b[:4] or a[4] == b[4] or (a[5] == RD and b[5] == RD):
            continue
        lo, hi = (a, b) if a[4] < b[4] else (b, a)
        cand = a[:4] + (lo[4], hi[4], lo[5], hi[5])
        if best is None or cand < best:
            best = cand
    return (1 if best is not None else 0), best


# --------------------------------------------------------------------------
# the five configs as hand-written loops (SURVEY.md §8d texts, transcribed)
# --------------------------------------------------------------------------
def loops_1a(B, M):
    out = []
    for tid in range(B):
        for x in range(M):
            out += [(0, 0, 0, x, tid, RD), (0, 0, 0, x, tid, WR)]
    return out


def loops_1b(B):
    return [(0, 0, 0, 0, 0, WR)] if B > 0 else []


def loops_2(variant, B):
    H, L = B // 2, B.bit_length() - 1
    out = []
    for tid in range(B):
        ph = 0
        out.append((ph, 0, 0, tid, tid, WR))
        if variant != "2c":
            ph += 1
        for k in range(L):
            s = H >> k
            if tid < s:
                out += [(ph, 0, 0, tid, tid, RD), (ph, 0, 0, tid + s, tid, RD), (ph, 0, 0, tid, tid, WR)]
            if variant != "2b":
                ph += 1
    return out


def loops_3(variant, TS, RW, G):
    out = []
    for b in range(G):
        for tid in range(TS * RW):
            for j in range(0, TS, RW):
                out.append((0, 0, b, (tid // TS + j) * TS + tid % TS, tid, WR))
            ph = 1 if variant == "3a" else 0
            for j in range(0, TS, RW):
                out.append((ph, 0, b, (tid % TS) * TS + tid // TS + j, tid, RD))
    return out


def loops_4ab(variant, N, BS):
    D = N.bit_length() - 1
    out = []
    for tid in range(BS):
        for d in range(D):
            for k in range(N // BS):
                e = k * BS + tid
                if variant == "4a":
                    cur, nxt = (d % 2) * N, ((d + 1) % 2) * N
                    if e >= (1 << d):
                        out += [(d, 0, 0, cur + e - (1 << d), tid, RD), (d, 0, 0, cur + e, tid, RD),
                                (d, 0, 0, nxt + e, tid, WR)]
                    else:
                        out += [(d, 0, 0, cur + e, tid, RD), (d, 0, 0, nxt + e, tid, WR)]
                else:
                    if e >= (1 << d):
                        out += [(d, 0, 0, e - (1 << d), tid, RD), (d, 0, 0, e, tid, RD), (d, 0, 0, e, tid, WR)]
    return out


def loops_4cd(variant, N, BS):
    D = N.bit_length() - 1
    out = []
    for tid in range(BS):
        ph = 0
        for k in range(N // BS):
            out.append((ph, 0, 0, k * BS + tid, tid, WR))
        ph += 1
        for l in range(D):                                   # up-sweep
            m = N >> (l + 1)
            for k in range((m + BS - 1) // BS):
                e = k * BS + tid
                if e < m:
                    ai, bi = (1 << l) * (2 * e + 1) - 1, (1 << l) * (2 * e + 2) - 1
                    out += [(ph, 0, 0, ai, tid, RD), (ph, 0, 0, bi, tid, RD), (ph, 0, 0, bi, tid, WR)]
            ph += 1
        if tid == 0:
            out.append((ph, 0, 0, N - 1, tid, WR))
        ph += 1
        for l in range(D):                                   # down-sweep
            s = N >> (l + 1)
            for k in range(((1 << l) + BS - 1) // BS):
                e = k * BS + tid
                if e < (1 << l):
                    ai, bi = s * (2 * e + 1) - 1, s * (2 * e + 2) - 1
                    out += [(ph, 0, 0, ai, tid, RD), (ph, 0, 0, bi, tid, RD), (ph, 0, 0, ai, tid, WR),
                            (ph, 0, 0, bi, tid, RD), (ph, 0, 0, bi, tid, WR)]
            if variant == "4c":
                ph += 1
    return out


def loops_5(variant, B, T, R, C):
    H = B * R
    out = []
    for tid in range(B):
        for t in range(T):
            cur = (t % 2) * H * C if variant == "5a" else 0
            nxt = ((t + 1) % 2) * H * C if variant == "5a" else 0
            for r in range(R):
                row = tid * R + r
                for c in range(C):
                    out += [(t, 0, 0, cur + ((row + H - 1) % H) * C + c, tid, RD),
                            (t, 0, 0, cur + row * C + c, tid, RD),
                            (t, 0, 0, cur + ((row + 1) % H) * C + c, tid, RD),
                            (t, 0, 0, nxt + row * C + c, tid, WR)]
    return out


def config_records(inst):
    """Hand-written loop version of a workloads.Instance (config families 1-5)."""
    name, p = inst.name, inst.params
    B = inst.n_threads
    if name == "1a":
        return loops_1a(B, p["M"])
    if name == "1b":
        return loops_1b(B)
    if name[0] == "2":
        return loops_2(name, B)
    if name[0] == "3":
        return loops_3(name, p["TS"], p["RW"], inst.n_blocks)
    if name in ("4a", "4b"):
        return loops_4ab(name, p["N"], p["BS"])
    if name in ("4c", "4d"):
        return loops_4cd(name, p["N"], p["BS"])
    if name[0] == "5":
        return loops_5(name, B, p["T"], p["R"], p["C"])
    raise KeyError(name)


# --------------------------------------------------------------------------
# direct evaluator of the fuzz AST (workloads/fuzz.py node shapes)
# --------------------------------------------------------------------------
class EvalError(Exception):
    pass


def _num(e, env):
    k = e[0]
    if k == "nat":
        return e[1]
    if k == "var":
        return env[e[1]]
    if k in ("tid", "bid"):
        return env[k]
    _, op, a, b = e
    x, y = _num(a, env), _num(b, env)
    if op == "+":
        return x + y
    if op == "-":
        return max(x - y, 0)                    # monus
    if op == "*":
        return x * y
    if op == "/":
        if y == 0:
            raise EvalError("div0")
        return x // y
    if op == "%":
        if y == 0:
            raise EvalError("div0")
        return x % y
    if op == "<<":
        return x << y
    if op == ">>":
        return x >> y
    if op == "min":
        return min(x, y)
    if op == "max":
        return max(x, y)
    raise ValueError(op)


def _cond(c, env):
    k = c[0]
    if k == "true":
        return True
    if k == "false":
        return False
    # DESIGN.md R2: both operands of and/or are evaluated (no short circuit), so a
    # division by zero in either operand is reached whenever the condition is
    if k == "and":
        x, y = _cond(c[1], env), _cond(c[2], env)
        return x and y
    if k == "or":
        x, y = _cond(c[1], env), _cond(c[2], env)
        return x or y
    _, op, a, b = c
    x, y = _num(a, env), _num(b, env)
    return {"=": x == y, "!=": x != y, "<": x < y, "<=": x <= y, ">": x > y, ">=": x >= y}[op]


def eval_ast(prog, grid, block, params):
    """Access records of a fuzz program (per-thread walk, union over threads)."""
    arrays = prog["arrays"]
    out = []
    nb = grid[0] * grid[1] * grid[2]
    nt = block[0] * block[1] * block[2]

    def run(s, env, st):
        k = s[0]
        if k == "skip":
            return
        if k == "sync":
            st["phase"] += 1
            return
        if k == "acc":
            out.append((st["phase"], arrays.index(s[2]), env["bid"], _num(s[3], env), env["tid"],
                        WR if s[1] == "wr" else RD))
            return
        if k == "seq":
            for x in s[1]:
                run(x, env, st)
            return
        if k == "if":
            run(s[2] if _cond(s[1], env) else s[3], env, st)
            return
        _, v, lo, hi, step, body = s
        a, b, d = _num(lo, env), _num(hi, env), _num(step, env)
        x = a
        while x < b:
            env2 = dict(env)
            env2[v] = x
            run(body, env2, st)
            x += d

    for bid in range(nb):
        for tid in range(nt):
            env = dict(params)
            env["tid"], env["bid"] = tid, bid
            run(prog["body"], env, {"phase": 0})
    return out
