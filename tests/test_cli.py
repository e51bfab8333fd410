"""The command line (python -m paper_2203_12878_b200) and its exit codes
(0 drf/ok, 1 racy, 2 ill-typed / unverified alarm, 3 parse error,
4 execution error, 5 Theorem-1 mismatch), on the paper's kernels in examples/."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(*args):
    r = subprocess.run([sys.executable, "-m", "paper_2203_12878_b200", *args, "--format", "json"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    return r.returncode, (json.loads(r.stdout.strip().splitlines()[-1]) if r.stdout.strip() else None), r.stderr


def test_typecheck_exit_codes():
    rc, rep, _ = cli("typecheck", "examples/racy.bcu")
    assert rc == 0 and rep["map"] == "params M; shared A; forU x in 0..M { rd A[x]; wr A[x] }"
    rc, rep, _ = cli("typecheck", "examples/drf.bcu")
    assert rc == 0 and rep["map"] == "shared A; if (tid = 0) { wr A[0] } else { skip }"
    rc, rep, _ = cli("typecheck", "examples/eq1.bcu")
    assert rc == 2 and rep["type_error"]["variable"] == "x" and rep["type_error"]["kind"] == "data_dependent_index"


def test_parse_error_exit_code(tmp_path):
    bad = tmp_path / "bad.bcu"
    bad.write_text("if (tid = 0) { A[0] := 1 }")          # BabyCUDA ifs need an else
    rc, rep, _ = cli("typecheck", str(bad))
    assert rc == 3 and "error" in rep


@pytest.mark.gpu
def test_check_run_verify_on_gpu():
    rc, rep, _ = cli("check", "examples/racy.bcu", "--threads", "2", "--set", "M=1")
    assert rc == 1 and rep["alarm"] == "true_alarm" and rep["witness"]["tid_hi"] == 1
    rc, rep, _ = cli("check", "examples/drf.bcu", "--threads", "8")
    assert rc == 0 and rep["verdict"] == "drf"
    rc, rep, _ = cli("check", "examples/eq1.bcu", "--threads", "2")
    assert rc == 2 and rep["alarm"] == "unverified_alarm"           # SPEC.md: check eq1.bcu -> exit 2
    rc, rep, _ = cli("run", "examples/eq1.bcu", "--threads", "8")
    assert rc == 0 and rep["verdict"] == "drf"                       # the execution itself has no race
    rc, rep, _ = cli("verify-theorem", "examples/racy.bcu", "--threads", "2", "--set", "M=2")
    assert rc == 0 and rep["equal"] and rep["access_values"] == 8    # SPEC.md: 8 access values
    rc, rep, _ = cli("verify-theorem", "examples/eq1.bcu", "--threads", "2")
    assert rc == 2
    rc, rep, _ = cli("check-map", "examples/racy.map", "--threads", "8", "--set", "M=8")
    assert rc == 1 and rep["n_accesses"] == 128
    rc, rep, _ = cli("run", "examples/reduce.bcu", "--threads", "1024", "--set", "H=512", "--set", "L=10")
    assert rc == 0 and rep["uninit_reads"] == 0
