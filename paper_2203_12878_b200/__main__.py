"""Command line: ``python -m paper_2203_12878_b200 SUBCOMMAND FILE [options]``.

Subcommands (the exit codes are SPEC.md:620's contract: 0 DRF / ok, 1 racy,
2 ill-typed or an unverified alarm, 3 parse / scope / barrier error, 4 execution
error, 5 Theorem-1 mismatch):

  check-map FILE       race-check a MAP (DESIGN.md §3 grammar) on the GPU
  typecheck FILE       type a BabyCUDA kernel (Fig. 6) and print its MAP
  check FILE           type it and race-check its MAP: a race on a typable kernel is a
                       TRUE alarm (Theorem 1); an ill-typed kernel is checked through its
                       data-abstracted MAP (--domain, default: its largest array extent),
                       whose alarms are unverified
  run FILE             execute the kernel with data on the GPU (Fig. 5) and race-check
                       the executed accesses
  verify-theorem FILE  executed access set == the inferred MAP's (Theorem 1)

Options: --grid X[,Y,Z] --block X[,Y,Z] (or --threads N) --set NAME=VALUE ... --domain D
--format human|json.  Every step runs in libmapcheck.so (no CPU fallback).
"""
from __future__ import annotations

import argparse
import json
import re
import sys

EXIT_DRF, EXIT_RACY, EXIT_TYPE, EXIT_PARSE, EXIT_EXEC, EXIT_MISMATCH = 0, 1, 2, 3, 4, 5
_INPUT_ERRORS = {1, 2, 3, 10}          # parse, scope, barrier, type


def _dims(text):
    v = [int(x) for x in text.split(",")]
    return tuple(v + [1] * (3 - len(v)))


def _args(argv):
    ap = argparse.ArgumentParser(prog="python -m paper_2203_12878_b200")
    ap.add_argument("command", choices=["check-map", "typecheck", "check", "run", "verify-theorem"])
    ap.add_argument("file")
    ap.add_argument("--grid", default="1")
    ap.add_argument("--block", default=None)
    ap.add_argument("--threads", type=int, default=None)
    ap.add_argument("--set", action="append", default=[], metavar="NAME=VALUE")
    ap.add_argument("--domain", type=int, default=0)
    ap.add_argument("--format", choices=["human", "json"], default="human")
    a = ap.parse_args(argv)
    a.grid = _dims(a.grid)
    a.block = _dims(a.block) if a.block else (a.threads or 1, 1, 1)
    a.params = {}
    for kv in a.set:
        name, _, val = kv.partition("=")
        a.params[name.strip()] = int(val)
    return a


def _witness(w):
    if w is None:
        return None
    return {"phase": w.phase, "array": w.array_name, "block": w.block, "index": w.index,
            "tid_lo": w.tid_lo, "kind_lo": "wr" if w.kind_lo else "rd",
            "tid_hi": w.tid_hi, "kind_hi": "wr" if w.kind_hi else "rd"}


def _emit(report, fmt, out=sys.stdout):
    if fmt == "json":
        out.write(json.dumps(report) + "\n")
        return
    for k, v in report.items():
        out.write(f"{k}: {v}\n")


def main(argv=None) -> int:
    a = _args(sys.argv[1:] if argv is None else argv)
    import paper_2203_12878_b200 as mc
    with open(a.file) as f:
        src = f.read()
    rep = {"command": a.command, "file": a.file}
    try:
        if a.command == "check-map":
            r = mc.MapProgram(src, a.grid, a.block, a.params).check_races()
            rep.update(verdict="racy" if r.verdict else "drf", witness=_witness(r.witness),
                       n_accesses=r.n_accesses, racy_cells=r.racy_segments)
            _emit(rep, a.format)
            return EXIT_RACY if r.verdict else EXIT_DRF
        inf = mc.infer(src)
        rep["typable"] = inf.typable
        if not inf.typable:
            rep["type_error"] = {"kind": inf.kind, "variable": inf.var, "line": inf.line, "col": inf.col}
        if a.command == "typecheck":
            rep["map"] = inf.map_text
            _emit(rep, a.format)
            return EXIT_DRF if inf.typable else EXIT_TYPE
        if a.command == "check":
            text = inf.map_text
            if not inf.typable:
                decl = re.search(r"\bshared\b([^;]*);", src)
                extents = [int(x) for x in re.findall(r"\[(\d+)\]", decl.group(1))] if decl else []
                dom = a.domain or max(extents or [a.block[0] * a.block[1] * a.block[2]])
                text = mc.infer(src, data_domain=dom).map_text
                rep["data_domain"] = dom
            r = mc.MapProgram(text, a.grid, a.block, a.params).check_races()
            rep.update(map=text, verdict="racy" if r.verdict else "drf", witness=_witness(r.witness),
                       n_accesses=r.n_accesses, racy_cells=r.racy_segments,
                       alarm=None if not r.verdict else ("true_alarm" if inf.typable else "unverified_alarm"))
            _emit(rep, a.format)
            if not r.verdict:
                return EXIT_DRF
            return EXIT_RACY if inf.typable else EXIT_TYPE
        k = mc.Kernel(src, a.grid, a.block, a.params)
        if a.command == "run":
            r = k.execute()
            rep.update(verdict="racy" if r.verdict else "drf", witness=_witness(r.witness), executed=r.n_events,
                       access_values=r.n_alpha, racy_cells=r.racy_segments, uninit_reads=r.uninit_reads,
                       ambiguous_reads=r.ambiguous_reads)
            _emit(rep, a.format)
            return EXIT_RACY if r.verdict else EXIT_DRF
        # verify-theorem
        if not inf.typable:
            _emit(rep, a.format)
            return EXIT_TYPE
        d = k.theorem1_diff(mc.MapProgram(inf.map_text, a.grid, a.block, a.params))
        rep.update(equal=d.equal, access_values=d.n_alpha, map_access_values=d.n_lambda,
                   only_executed=d.only_alpha, only_map=d.only_lambda)
        _emit(rep, a.format)
        return EXIT_DRF if d.equal else EXIT_MISMATCH
    except mc.MapError as e:
        rep["error"] = str(e)
        _emit(rep, a.format)
        return EXIT_PARSE if e.status in _INPUT_ERRORS else EXIT_EXEC


if __name__ == "__main__":
    sys.exit(main())
