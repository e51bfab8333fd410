"""The CPU oracle's throughput on configs 1-4 at full size (all host
cores and one thread), for context next to the GPU numbers (bench.py other_configs)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from workloads import config

cores = os.cpu_count() or 1
for name in ("1a", "1b", "2a", "2b", "2c", "3a", "3b", "4a", "4b", "4c", "4d"):
    inst = config(name)
    out = {"cfg": name, "cores": cores}
    for th in (1, cores):
        t0 = time.perf_counter()
        r = oracle.check_instance(inst, threads=th)
        dt = time.perf_counter() - t0
        out[f"threads_{th}"] = {"s": round(dt, 4), "G_acc_s": round(r.n_accesses / dt / 1e9, 4)}
    out["n_accesses"] = r.n_accesses
    out["verdict"] = "racy" if r.verdict else "drf"
    print(json.dumps(out), flush=True)
