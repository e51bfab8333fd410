"""BabyCUDA oracle -- TEST INFRASTRUCTURE (plain, slow, obviously correct).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import this
module; the product path (paper_2203_12878_b200) never does and shares no code
with it.  It follows arxiv 2203.12878 rule by rule:

* ``infer``   -- the behavioural type system of Fig. 6 (prose
  :803-834): rules t-n, t-b, t-write, t-read, t-seq, t-if, t-for, t-skip, under
  the context V = {tid, bid} u params; a kernel that indexes or branches on a
  value read from an array is ill-typed (Eq. 1).  Extended to
  the synchronized fragment ("extends easily"): sync types to sync,
  a loop whose body contains sync types to forS (R18).
* ``execute`` -- the big-step semantics of Fig. 5: rules read
  (a thread sees lastwrite over its own current-phase record consed onto the
  history, so its own in-phase writes and earlier phases' writes),
  write (W[y -> z]), seq, if-t/if-f, for-1/for-2, skip, and par (every thread
  runs from the same history; the phase is the union of their records,
  PAPER.md:579-589); lastwrite-curr / -prev / -undef.
  ``sync`` closes the phase of every thread of the block (R18).
* ``alpha``  -- the access values of a phase, alpha in^ P:
  (i, rd, y) for y in R, (i, wr, y) for y in dom(W).

Readings (R18-R24): per-block arrays (R10); naturals are exact
u64 -- an operation whose exact result exceeds 2^64 - 1 is a range error (R3),
x / 0 and x % 0 are arithmetic errors (R4); lastwrite-undef (bottom) reads as 0
and is counted (R20); when several threads of the consulted phase wrote the
index, lastwrite takes the value of the smallest such tid and the read is
counted as ambiguous (R21); an index at or beyond the array's declared extent
is a range error (R22).

The race check of the executed phases uses the paper's definition directly
(PAPER.md:111-113): two accesses of one (phase, array, block, index) by distinct
threads, at least one a write; witness = lexicographic minimum (R14).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

U64 = (1 << 64) - 1
RD, WR = 0, 1

S_OK, S_PARSE, S_SCOPE, S_BARRIER, S_RANGE, S_ARITH, S_ARG, S_TYPE = 0, 1, 2, 3, 4, 5, 8, 10
T_OK, T_DATA_INDEX, T_DATA_CONTROL = 0, 1, 2          # ill-typed kinds (first failing premise)

KEYWORDS = {"params", "shared", "skip", "sync", "let", "in", "if", "else", "for", "step", "true", "false",
            "and", "or", "min", "max", "tid", "bid"}


class BcError(Exception):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


# ============================================================== lexer ======
def _lex(src: str):
    toks, i, line, col = [], 0, 1, 1
    two = {":=", "..", "<=", ">=", "!=", "<<", ">>"}
    while i < len(src):
        c = src[i]
        if c == "\n":
            i, line, col = i + 1, line + 1, 1
            continue
        if c in " \t\r":
            i, col = i + 1, col + 1
            continue
        if src.startswith("//", i):
            while i < len(src) and src[i] != "\n":
                i += 1
            continue
        if c.isdigit():
            j = i
            while j < len(src) and src[j].isdigit():
                j += 1
            v = int(src[i:j])
            if v > U64:
                raise BcError(S_RANGE, f"{line}:{col}: literal too large")
            toks.append(("nat", v, line, col))
        elif c.isalpha() or c == "_":
            j = i
            while j < len(src) and (src[j].isalnum() or src[j] == "_"):
                j += 1
            w = src[i:j]
            toks.append(("kw" if w in KEYWORDS else "id", w, line, col))
        elif src[i:i + 2] in two:
            j = i + 2
            toks.append(("op", src[i:j], line, col))
        elif c in "+-*/%<>=(){}[];,":
            j = i + 1
            toks.append(("op", c, line, col))
        else:
            raise BcError(S_PARSE, f"{line}:{col}: unexpected character {c!r}")
        col += j - i
        i = j
    toks.append(("eof", None, line, col))
    return toks


# ============================================================= parser ======
# AST (tuples; every node carries (line, col) as its last element):
#   num : ("nat", v, pos) | ("var", name, pos) | ("tid", pos) | ("bid", pos) | ("bin", op, a, b, pos)
#   cond: ("true", pos) | ("false", pos) | ("rel", op, a, b, pos) | ("and", l, r, pos) | ("or", l, r, pos)
#   stmt: ("skip", pos) | ("sync", pos) | ("write", arr, idx, payload, pos)
#         | ("let", var, arr, idx, body, pos) | ("if", cond, then, else, pos)
#         | ("for", var, lo, hi, step, body, pos) | ("seq", [stmts], pos)
class _Parser:
    def __init__(self, src):
        self.t = _lex(src)
        self.i = 0

    def peek(self, k=0):
        return self.t[self.i + k]

    def pos(self):
        return (self.peek()[2], self.peek()[3])

    def is_(self, v):
        return self.peek()[1] == v and self.peek()[0] in ("op", "kw")

    def eat(self, v):
        if not self.is_(v):
            tk = self.peek()
            raise BcError(S_PARSE, f"{tk[2]}:{tk[3]}: expected {v!r}, got {tk[1]!r}")
        self.i += 1

    def ident(self):
        tk = self.peek()
        if tk[0] != "id":
            raise BcError(S_PARSE, f"{tk[2]}:{tk[3]}: expected an identifier, got {tk[1]!r}")
        self.i += 1
        return tk[1]

    def nat(self):
        tk = self.peek()
        if tk[0] != "nat":
            raise BcError(S_PARSE, f"{tk[2]}:{tk[3]}: expected a natural number")
        self.i += 1
        return tk[1]

    # numeric expressions: shifts < additive < multiplicative < atoms (left-assoc)
    def num(self):
        a = self.additive()
        while self.is_("<<") or self.is_(">>"):
            p = self.pos()
            op = self.peek()[1]
            self.i += 1
            a = ("bin", op, a, self.additive(), p)
        return a

    def additive(self):
        a = self.mult()
        while self.is_("+") or self.is_("-"):
            p = self.pos()
            op = self.peek()[1]
            self.i += 1
            a = ("bin", op, a, self.mult(), p)
        return a

    def mult(self):
        a = self.atom()
        while self.is_("*") or self.is_("/") or self.is_("%"):
            p = self.pos()
            op = self.peek()[1]
            self.i += 1
            a = ("bin", op, a, self.atom(), p)
        return a

    def atom(self):
        tk = self.peek()
        p = (tk[2], tk[3])
        if tk[0] == "nat":
            self.i += 1
            return ("nat", tk[1], p)
        if tk[0] == "id":
            self.i += 1
            return ("var", tk[1], p)
        if self.is_("tid"):
            self.i += 1
            return ("tid", p)
        if self.is_("bid"):
            self.i += 1
            return ("bid", p)
        if self.is_("min") or self.is_("max"):
            op = tk[1]
            self.i += 1
            self.eat("(")
            a = self.num()
            self.eat(",")
            b = self.num()
            self.eat(")")
            return ("bin", op, a, b, p)
        if self.is_("("):
            self.i += 1
            a = self.num()
            self.eat(")")
            return a
        raise BcError(S_PARSE, f"{tk[2]}:{tk[3]}: expected an expression, got {tk[1]!r}")

    # conditions: or < and < atoms; "(" is ambiguous (condition or expression): backtrack
    def cond(self):
        a = self.cand()
        while self.is_("or"):
            p = self.pos()
            self.i += 1
            a = ("or", a, self.cand(), p)
        return a

    def cand(self):
        a = self.catom()
        while self.is_("and"):
            p = self.pos()
            self.i += 1
            a = ("and", a, self.catom(), p)
        return a

    def catom(self):
        p = self.pos()
        if self.is_("true"):
            self.i += 1
            return ("true", p)
        if self.is_("false"):
            self.i += 1
            return ("false", p)
        if self.is_("("):
            save = self.i
            try:
                self.i += 1
                c = self.cond()
                self.eat(")")
                return c
            except BcError:
                self.i = save
        a = self.num()
        for op in ("=", "!=", "<=", ">=", "<", ">"):
            if self.is_(op):
                self.i += 1
                return ("rel", op, a, self.num(), p)
        tk = self.peek()
        raise BcError(S_PARSE, f"{tk[2]}:{tk[3]}: expected a comparison")

    # statements; `let y = A[n] in` takes the rest of the enclosing block as its body
    def block(self, stop):
        p = self.pos()
        items = []
        while True:
            if self.is_("let"):
                items.append(self.let_stmt())
                break
            items.append(self.stmt())
            if self.is_(";"):
                self.i += 1
                if self.peek()[0] == "eof" or self.is_(stop):
                    break
                continue
            break
        return items[0] if len(items) == 1 else ("seq", items, p)

    def let_stmt(self):
        p = self.pos()
        self.eat("let")
        y = self.ident()
        self.eat("=")
        arr = self.ident()
        self.eat("[")
        idx = self.num()
        self.eat("]")
        self.eat("in")
        body = self.block("}")
        return ("let", y, arr, idx, body, p)

    def stmt(self):
        p = self.pos()
        if self.is_("skip"):
            self.i += 1
            return ("skip", p)
        if self.is_("sync"):
            self.i += 1
            return ("sync", p)
        if self.is_("if"):
            self.i += 1
            self.eat("(")
            c = self.cond()
            self.eat(")")
            self.eat("{")
            t = self.block("}")
            self.eat("}")
            self.eat("else")          # BabyCUDA conditionals always have an else
            self.eat("{")
            e = self.block("}")
            self.eat("}")
            return ("if", c, t, e, p)
        if self.is_("for"):
            self.i += 1
            x = self.ident()
            self.eat("in")
            lo = self.num()
            self.eat("..")
            hi = self.num()
            st = ("nat", 1, p)
            if self.is_("step"):
                self.i += 1
                st = self.num()
            self.eat("{")
            body = self.block("}")
            self.eat("}")
            return ("for", x, lo, hi, st, body, p)
        if self.peek()[0] == "id":
            arr = self.ident()
            self.eat("[")
            idx = self.num()
            self.eat("]")
            self.eat(":=")
            return ("write", arr, idx, self.num(), p)
        tk = self.peek()
        raise BcError(S_PARSE, f"{tk[2]}:{tk[3]}: expected a statement, got {tk[1]!r}")


@dataclass
class Kernel:
    params: List[str]
    arrays: List[str]
    extents: Dict[str, Optional[int]]
    body: tuple


def parse(src: str) -> Kernel:
    """Parse BabyCUDA text (grammar: DESIGN.md §3b) and resolve names."""
    ps = _Parser(src)
    params, arrays, extents = [], [], {}
    while ps.is_("params") or ps.is_("shared"):
        if ps.is_("params"):
            ps.i += 1
            params.append(ps.ident())
            while ps.is_(","):
                ps.i += 1
                params.append(ps.ident())
        else:
            ps.i += 1
            while True:
                a = ps.ident()
                arrays.append(a)
                extents[a] = None
                if ps.is_("["):
                    ps.i += 1
                    extents[a] = ps.nat()
                    ps.eat("]")
                if not ps.is_(","):
                    break
                ps.i += 1
        ps.eat(";")
    body = ps.block(None)
    if ps.peek()[0] != "eof":
        tk = ps.peek()
        raise BcError(S_PARSE, f"{tk[2]}:{tk[3]}: unexpected {tk[1]!r}")
    if not arrays:                      # the paper's single array A
        arrays, extents = ["A"], {"A": None}
    if len(set(params + arrays)) != len(params) + len(arrays):
        raise BcError(S_SCOPE, "duplicate parameter or array name")
    k = Kernel(params, arrays, extents, body)
    _resolve(k)
    _check_barriers(k)
    return k


def _check_barriers(k: Kernel):
    """R8 for kernels: a sync is never under an if, and a loop around a sync has
    bounds that are the same for every thread of the block (no tid, no value read
    from an array) -- otherwise threads could disagree on the barrier sequence."""
    def go(s, under_if, data):
        t = s[0]
        if t == "sync" and under_if:
            raise BcError(S_BARRIER, f"{s[1][0]}:{s[1][1]}: sync under a conditional")
        if t == "let":
            go(s[4], under_if, data | {s[1]})
        elif t == "if":
            go(s[2], True, data)
            go(s[3], True, data)
        elif t == "for":
            if _has_sync(s[5]):
                for e in s[2:5]:
                    for x, pos in free_vars(e):
                        if x in ("tid", "bid") or x in data:
                            raise BcError(S_BARRIER, f"{pos[0]}:{pos[1]}: loop around a sync depends on {x}")
            go(s[5], under_if, data)
        elif t == "seq":
            for x in s[1]:
                go(x, under_if, data)
    go(k.body, False, frozenset())


def _resolve(k: Kernel):
    """Scope check: every variable bound; binders distinct from every name in
    scope (the paper requires distinct nested binders)."""
    def num(e, scope):
        if e[0] == "var" and e[1] not in scope:
            raise BcError(S_SCOPE, f"{e[2][0]}:{e[2][1]}: unbound variable {e[1]}")
        if e[0] == "bin":
            num(e[2], scope)
            num(e[3], scope)

    def cond(c, scope):
        if c[0] == "rel":
            num(c[2], scope)
            num(c[3], scope)
        elif c[0] in ("and", "or"):
            cond(c[1], scope)
            cond(c[2], scope)

    def bind(x, scope, pos):
        if x in scope or x in k.arrays:
            raise BcError(S_SCOPE, f"{pos[0]}:{pos[1]}: binder {x} shadows a name in scope")
        return scope | {x}

    def stmt(s, scope):
        t = s[0]
        if t == "write":
            if s[1] not in k.arrays:
                raise BcError(S_SCOPE, f"{s[4][0]}:{s[4][1]}: unknown array {s[1]}")
            num(s[2], scope)
            num(s[3], scope)
        elif t == "let":
            if s[2] not in k.arrays:
                raise BcError(S_SCOPE, f"{s[5][0]}:{s[5][1]}: unknown array {s[2]}")
            num(s[3], scope)
            stmt(s[4], bind(s[1], scope, s[5]))
        elif t == "if":
            cond(s[1], scope)
            stmt(s[2], scope)
            stmt(s[3], scope)
        elif t == "for":
            for e in (s[2], s[3], s[4]):
                num(e, scope)
            stmt(s[5], bind(s[1], scope, s[6]))
        elif t == "seq":
            for x in s[1]:
                stmt(x, scope)

    stmt(k.body, frozenset(k.params))


# ============================================================ typing =======
def free_vars(e) -> List[Tuple[str, tuple]]:
    """FV(n) / FV(c) in left-to-right order, with positions (tid/bid count as variables)."""
    t = e[0]
    if t == "var":
        return [(e[1], e[2])]
    if t in ("tid", "bid"):
        return [(t, e[1])]
    if t == "bin":
        return free_vars(e[2]) + free_vars(e[3])
    if t == "rel":
        return free_vars(e[2]) + free_vars(e[3])
    if t in ("and", "or"):
        return free_vars(e[1]) + free_vars(e[2])
    return []


@dataclass
class Typing:
    typable: bool
    protocol: Optional[tuple] = None      # MAP AST (see map_text) when typable
    kind: int = T_OK                      # T_DATA_INDEX / T_DATA_CONTROL
    var: str = ""
    line: int = 0
    col: int = 0


class _IllTyped(Exception):
    def __init__(self, kind, var, pos):
        self.kind, self.var, self.pos = kind, var, pos


def _has_sync(s) -> bool:
    t = s[0]
    if t == "sync":
        return True
    if t == "seq":
        return any(_has_sync(x) for x in s[1])
    if t == "let":
        return _has_sync(s[4])
    if t == "if":
        return _has_sync(s[2]) or _has_sync(s[3])
    if t == "for":
        return _has_sync(s[5])
    return False


def _t_expr(V, e, kind):
    """t-n / t-b: FV(e) subset of V, else the first offending variable."""
    for (x, pos) in free_vars(e):
        if x not in V:
            raise _IllTyped(kind, x, pos)


def _u_infer(V, b):
    """V |- b => u  (Fig. 6).  MAP AST: ("acc", o, arr, n) | ("seq", [..]) | ("if", c, u1, u2)
    | ("forU"|"forS", x, lo, hi, step, u) | ("skip",) | ("sync",)."""
    t = b[0]
    if t == "skip":                                    # t-skip
        return ("skip",)
    if t == "sync":                                    # synchronized extension (R18)
        return ("sync",)
    if t == "write":                                   # t-write: V |- n  =>  wr[n]   (payload erased)
        _t_expr(V, b[2], T_DATA_INDEX)
        return ("acc", WR, b[1], b[2])
    if t == "let":                                     # t-read: V |- n, y not in V, V |- b => u  =>  rd[n]; u
        _t_expr(V, b[3], T_DATA_INDEX)
        assert b[1] not in V                           # guaranteed by _resolve (distinct binders)
        u = _u_infer(V, b[4])                          # NOTE: y is NOT added to V
        return ("seq", [("acc", RD, b[2], b[3]), u])
    if t == "seq":                                     # t-seq
        return ("seq", [_u_infer(V, x) for x in b[1]])
    if t == "if":                                      # t-if
        _t_expr(V, b[1], T_DATA_CONTROL)
        return ("if", b[1], _u_infer(V, b[2]), _u_infer(V, b[3]))
    if t == "for":                                     # t-for: V |- n, V |- m, x not in V, V u {x} |- b => u
        for e in (b[2], b[3], b[4]):
            _t_expr(V, e, T_DATA_CONTROL)
        u = _u_infer(V | {b[1]}, b[5])
        return ("forS" if _has_sync(b[5]) else "forU", b[1], b[2], b[3], b[4], u)
    raise AssertionError(t)


def infer(k: Kernel) -> Typing:
    """Type the kernel under V = {tid, bid} u params (Theorem 1 uses {tid})."""
    V = frozenset(["tid", "bid"] + k.params)
    try:
        return Typing(True, _u_infer(V, k.body))
    except _IllTyped as e:
        return Typing(False, None, e.kind, e.var, e.pos[0], e.pos[1])


def abstract_protocol(k: Kernel, domain: int):
    """The MAP of an ill-typed kernel with array data abstracted (Faial's view,
    PAPER.md:880-885): a read whose value reaches an index, a condition or a loop
    bound becomes rd[n]; forU y in 0..domain { u } -- the accesses the thread
    makes for every value y it could have read in [0, domain).  Returns a MAP AST."""
    def uses(s, y) -> bool:                 # y in a typed position (index, condition, loop bound) of s
        data = {y}

        def go(s, data):
            t = s[0]
            if t == "write":
                return any(x in data for x, _ in free_vars(s[2]))
            if t == "let":
                if any(x in data for x, _ in free_vars(s[3])):
                    return True
                return go(s[4], data)
            if t == "if":
                return any(x in data for x, _ in free_vars(s[1])) or go(s[2], data) or go(s[3], data)
            if t == "for":
                return any(x in data for e in s[2:5] for x, _ in free_vars(e)) or go(s[5], data)
            if t == "seq":
                return any(go(x, data) for x in s[1])
            return False
        return go(s, data)

    def conv(b):
        t = b[0]
        if t in ("skip", "sync"):
            return (t,)
        if t == "write":
            return ("acc", WR, b[1], b[2])
        if t == "let":
            u = conv(b[4])
            if uses(b[4], b[1]):
                u = ("forU", b[1], ("nat", 0, b[5]), ("nat", domain, b[5]), ("nat", 1, b[5]), u)
            return ("seq", [("acc", RD, b[2], b[3]), u])
        if t == "seq":
            return ("seq", [conv(x) for x in b[1]])
        if t == "if":
            return ("if", b[1], conv(b[2]), conv(b[3]))
        if t == "for":
            return ("forS" if _has_sync(b[5]) else "forU", b[1], b[2], b[3], b[4], conv(b[5]))
        raise AssertionError(t)
    return conv(k.body)


def _num_text(e) -> str:
    t = e[0]
    if t == "nat":
        return str(e[1])
    if t == "var":
        return e[1]
    if t in ("tid", "bid"):
        return t
    op, a, b = e[1], _num_text(e[2]), _num_text(e[3])
    if op in ("min", "max"):
        return f"{op}({a}, {b})"
    return f"({a} {op} {b})"


def _cond_text(c) -> str:
    t = c[0]
    if t in ("true", "false"):
        return t
    if t == "rel":
        return f"{_num_text(c[2])} {c[1]} {_num_text(c[3])}"
    return f"({_cond_text(c[1])} {t} {_cond_text(c[2])})"


def map_text(k: Kernel, proto) -> str:
    """Print a MAP AST in the MAP grammar of DESIGN.md §3 (fully parenthesised)."""
    def go(u) -> str:
        t = u[0]
        if t in ("skip", "sync"):
            return t
        if t == "acc":
            return f"{'wr' if u[1] == WR else 'rd'} {u[2]}[{_num_text(u[3])}]"
        if t == "seq":
            return "; ".join(go(x) for x in u[1])
        if t == "if":
            return f"if ({_cond_text(u[1])}) {{ {go(u[2])} }} else {{ {go(u[3])} }}"
        step = "" if u[4][0] == "nat" and u[4][1] == 1 else f" step {_num_text(u[4])}"
        return f"{t} {u[1]} in {_num_text(u[2])}..{_num_text(u[3])}{step} {{ {go(u[5])} }}"
    head = (f"params {', '.join(k.params)}; " if k.params else "") + f"shared {', '.join(k.arrays)}; "
    return head + go(proto)


# ========================================================= semantics =======
def _ev(e, env) -> int:
    """n => y over naturals, exact u64 (R3, R4)."""
    t = e[0]
    if t == "nat":
        return e[1]
    if t == "var":
        return env[e[1]]
    if t in ("tid", "bid"):
        return env[t]
    op = e[1]
    a, b = _ev(e[2], env), _ev(e[3], env)
    if op == "+":
        r = a + b
    elif op == "-":
        r = a - b if a > b else 0                    # monus
    elif op == "*":
        r = a * b
    elif op in ("/", "%"):
        if b == 0:
            raise BcError(S_ARITH, f"{e[4][0]}:{e[4][1]}: division by zero")
        r = a // b if op == "/" else a % b
    elif op == "<<":
        r = 0 if a == 0 else (a << b if b < 64 else U64 + 1)
    elif op == ">>":
        r = a >> b if b < 64 else 0
    elif op == "min":
        r = min(a, b)
    else:
        r = max(a, b)
    if r > U64:
        raise BcError(S_RANGE, f"{e[4][0]}:{e[4][1]}: value exceeds 64 bits")
    return r


def _cv(c, env) -> bool:
    t = c[0]
    if t == "true":
        return True
    if t == "false":
        return False
    if t in ("and", "or"):                            # R2: both operands evaluated
        x, y = _cv(c[1], env), _cv(c[2], env)
        return (x and y) if t == "and" else (x or y)
    a, b = _ev(c[2], env), _ev(c[3], env)
    return {"=": a == b, "!=": a != b, "<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b}[c[1]]


@dataclass
class Counters:
    uninit: int = 0
    ambiguous: int = 0


def lastwrite(y, history, counters: Optional[Counters] = None):
    """lastwrite_y(H): the value of the most recent phase whose
    records write y (lastwrite-curr), skipping phases that do not (lastwrite-prev);
    None = bottom for the empty history (lastwrite-undef).  history: newest first;
    a phase maps tid -> (R, W).  Several writers in the consulted phase: the
    smallest tid's value (R21)."""
    for P in history:
        writers = sorted(i for i, (_, W) in P.items() if y in W)
        if writers:
            if len(writers) > 1 and counters is not None:
                counters.ambiguous += 1
            return P[writers[0]][1][y]
        # lastwrite-prev: no record of this phase has y in dom(W)
    return None                                        # lastwrite-undef


def _thread(k: Kernel, s, env, rec, hist_of, extents, emit, counters):
    """<A> b => B for one thread (Fig. 5) as a generator that yields at every sync;
    rec = [R, W] of the current phase (mutated in place; the driver swaps it at sync)."""
    t = s[0]
    if t == "skip":                                                   # skip
        return
    if t == "sync":
        yield "sync"
        return
    if t == "write":                                                  # write: n => y, m => z
        arr = s[1]
        y = _ev(s[2], env)
        z = _ev(s[3], env)
        _bound(arr, y, extents, s[4])
        rec[0][1][(arr, y)] = z                                       # W[y -> z]
        emit(arr, y, WR)
        return
    if t == "let":                                                    # read
        arr = s[2]
        y = _ev(s[3], env)
        _bound(arr, y, extents, s[5])
        rec[0][0].add((arr, y))                                       # R u {y}
        emit(arr, y, RD)
        # lastwrite_y({i : (R, W)} :: H): the thread's own current record first
        own = {env["tid"]: (rec[0][0], rec[0][1])}
        v = lastwrite((arr, y), [own] + hist_of(), counters)
        if v is None:
            counters.uninit += 1
            v = 0                                                     # R20
        env2 = dict(env)
        env2[s[1]] = v                                                # b[v / x]
        yield from _thread(k, s[4], env2, rec, hist_of, extents, emit, counters)
        return
    if t == "seq":                                                    # seq
        for x in s[1]:
            yield from _thread(k, x, env, rec, hist_of, extents, emit, counters)
        return
    if t == "if":                                                     # if-t / if-f
        branch = s[2] if _cv(s[1], env) else s[3]
        yield from _thread(k, branch, env, rec, hist_of, extents, emit, counters)
        return
    if t == "for":                                                    # for-1 / for-2
        lo, hi, st = _ev(s[2], env), _ev(s[3], env), _ev(s[4], env)
        if st == 0:                                                   # as the MAP oracle (R6)
            raise BcError(S_ARITH, f"{s[6][0]}:{s[6][1]}: loop step is zero")
        x = lo
        while x < hi:                                                 # for-2: n < m
            env2 = dict(env)
            env2[s[1]] = x                                            # b[n / x]
            yield from _thread(k, s[5], env2, rec, hist_of, extents, emit, counters)
            x += st                                                   # for lo+1 .. m (stride R6)
        return                                                        # for-1: n >= m
    raise AssertionError(t)


def _bound(arr, y, extents, pos):
    e = extents.get(arr)
    if e is not None and y >= e:
        raise BcError(S_RANGE, f"{pos[0]}:{pos[1]}: index {y} outside {arr}[{e}]")


@dataclass
class ExecResult:
    status: int = 0
    diag: str = ""
    n_events: int = 0                       # accesses executed (multiset)
    alpha: frozenset = frozenset()          # {(phase, array, block, index, tid, kind)}: alpha in^ P, all phases
    verdict: int = 0
    witness: Optional[tuple] = None
    racy_segments: int = 0
    uninit_reads: int = 0
    ambiguous_reads: int = 0
    n_phases: int = 0
    memory: Optional[list] = None           # [block][array] -> {index: value} of lastwrite over the history
    history: Optional[list] = None          # [block] -> phases oldest first, tid -> (R, W) over (array, index)


def execute(src: str, grid=(1, 1, 1), block=(1, 1, 1), params: Optional[Dict[str, int]] = None,
            thread_order: Optional[Sequence[int]] = None, keep_memory: bool = False,
            keep_history: bool = False) -> ExecResult:
    """Run the kernel on every block (rule par per phase) and check the executed
    phases for races.  thread_order permutes the order threads are run in (the
    result must not depend on it: par has no inter-thread premise)."""
    params = dict(params or {})
    try:
        k = parse(src)
        for p in k.params:
            if p not in params:
                raise BcError(S_ARG, f"missing parameter {p}")
        nb = grid[0] * grid[1] * grid[2]
        nt = block[0] * block[1] * block[2]
        order = list(thread_order) if thread_order is not None else list(range(nt))
        counters = Counters()
        events = []
        memory = [] if keep_memory else None
        histories = [] if keep_history else None
        n_phases = 1
        arr_id = {a: i for i, a in enumerate(k.arrays)}
        for b in range(nb):
            history: List[dict] = []                 # newest first
            phase = [0]
            gens, recs = {}, {}
            for i in order:
                env = dict(params)
                env.update(tid=i, bid=b)
                rec = [(set(), {})]
                recs[i] = rec

                def emit(arr, y, o, i=i):
                    events.append((phase[0], arr_id[arr], b, y, i, o))
                gens[i] = _thread(k, k.body, env, rec, lambda: history, k.extents, emit, counters)
            alive = list(order)
            while alive:
                at_sync, done = [], []
                for i in alive:                      # every thread up to its next sync (or the end)
                    try:
                        next(gens[i])
                        at_sync.append(i)
                    except StopIteration:
                        done.append(i)
                if at_sync and done:
                    raise BcError(S_BARRIER, "barrier divergence: some threads reached a sync, others ended")
                P = {i: recs[i][0] for i in order}   # rule par: the phase is every thread's record
                history.insert(0, P)
                for i in order:
                    recs[i][0] = (set(), {})
                alive = at_sync
                if at_sync:
                    phase[0] += 1
            n_phases = max(n_phases, phase[0] + 1)
            if keep_history:
                histories.append(list(reversed(history)))
            if keep_memory:
                mem = []
                for a in k.arrays:
                    cells = {y for P in history for (_, W) in P.values() for (aa, y) in W if aa == a}
                    mem.append({y: lastwrite((a, y), history) for y in sorted(cells)})
                memory.append(mem)
        alpha = frozenset(events)
        out = ExecResult(n_events=len(events), alpha=alpha, uninit_reads=counters.uninit,
                         ambiguous_reads=counters.ambiguous, n_phases=n_phases, memory=memory,
                         history=histories)
        out.verdict, out.witness, out.racy_segments = races(alpha)
        return out
    except BcError as e:
        return ExecResult(status=e.status, diag=str(e))


def races(accesses) -> Tuple[int, Optional[tuple], int]:
    """Race definition over a set of (phase, array, block, index, tid, kind):
    (verdict, canonical witness (phase, array, block, index, t_lo, t_hi, k_lo, k_hi), racy cells)."""
    cells: Dict[tuple, list] = {}
    for (ph, a, b, y, i, o) in accesses:
        cells.setdefault((ph, a, b, y), []).append((i, o))
    best, n = None, 0
    for cell, lst in cells.items():
        racy = False
        for (i1, o1), (i2, o2) in itertools.combinations(sorted(set(lst)), 2):
            if i1 != i2 and (o1 == WR or o2 == WR):
                lo, hi = ((i1, o1), (i2, o2)) if (i1, o1) < (i2, o2) else ((i2, o2), (i1, o1))
                w = cell + (lo[0], hi[0], lo[1], hi[1])
                best = w if best is None or w < best else best
                racy = True
        n += racy
    return (1 if best else 0), best, n


def infer_text(src: str, domain: int = 0) -> Tuple[int, Typing, str]:
    """(status, typing, MAP text): the inferred MAP of a typable kernel; for an
    ill-typed one the data-abstracted MAP when domain > 0, else status S_TYPE."""
    try:
        k = parse(src)
    except BcError as e:
        return e.status, Typing(False), ""
    ty = infer(k)
    if ty.typable:
        return S_OK, ty, map_text(k, ty.protocol)
    if domain > 0:
        return S_OK, ty, map_text(k, abstract_protocol(k, domain))
    return S_TYPE, ty, ""
