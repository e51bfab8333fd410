"""bench.py's multi-GPU entry point on CPU: `--gpus N` without a torchrun
environment re-launches the script as N ranks (torch.distributed.run, gloo for
the reference arm), and the JSON line reports them."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    env["OMP_NUM_THREADS"] = "2"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    return lines


def test_bench_gpus2_relaunches_two_ranks():
    lines = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-rows", "1"])
    assert len(lines) == 1                      # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["ranks"] == 2
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"


def test_bench_world_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr
