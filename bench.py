#!/usr/bin/env python
"""bench.py -- G accesses checked/s of the concrete MAP race check on B200.

Workload (BASELINE.json configs[4], the metric's headline config): the
synthetic 3-deep loop stencil MAP of SURVEY.md §8d, 2^34 accesses
(blockDim 1024, T=16 barrier phases, R=256 rows/thread, C=1024 columns,
ping-pong buffers -> DRF), checked exhaustively: one step = generate + radix
(detect path chosen per chunk) over every access of every phase.
The detect path is the library's automatic choice (for 5a: the sort-free
direct-address table, SURVEY.md §8f NEXT-3 -- every access folded into its
cell with one atomic OR, the table scanned once; no key is materialised and
nothing is sorted); `--detect table|sort` forces
the bucket-table path (partial LSD sort + shared-memory tables) or the full LSD
sort + segmented scan (the north_star's generate -> sort -> detect), and the
line also reports both of those paths' throughput on the same run
("detect_paths") and the radix pass's roofline ("roofline_sort_path").

Contract: `python bench.py --gpus N --steps K --warmup W` (one rank per GPU;
for N>1 under torchrun, or, when started without WORLD_SIZE, bench.py
re-launches itself under torch.distributed.run with N processes).  The plan is
cut into >= 2 chunks per rank (map_default_chunk) and every rank runs a
contiguous, bound-balanced range of chunks (map_rank_chunks) with no data-path
collective -- strong scaling on the fixed 2^34-access workload; `--mode
exchange` instead runs the north_star's key exchange (hash-bucketed generate ->
NCCL all_to_all -> local sort + detect).  Rank 0 prints ONE JSON line.  `--impl reference`
times the CPU oracle (the only reference this paper has) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import config  # noqa: E402

METRIC = "G accesses checked/s"
UNIT = "G accesses/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="5a")
    ap.add_argument("--chunk", type=int, default=0, help="chunk_max_accesses (0 = library default, 2^30)")
    ap.add_argument("--cpu-rows", type=int, default=64, help="R of the oracle's bounded sample (cpu_baseline leg)")
    ap.add_argument("--ref-rows", type=int, default=16,
                    help="R of the oracle's bounded sample per step of --impl reference (K+W steps must fit minutes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--detect", choices=["auto", "direct", "sort", "table"], default="auto")
    ap.add_argument("--no-alt-path", action="store_true", help="skip timing the other detect paths")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip timing the other BASELINE.json config families (context, not the metric)")
    ap.add_argument("--plain-scratch", action="store_true",
                    help="scratch in plain device memory (torch.empty) instead of map_scratch_alloc's compressible memory")
    ap.add_argument("--mode", choices=["shard", "exchange"], default="shard",
                    help="multi-GPU mode: chunk sharding (default) or the key exchange (all_to_all)")
    return ap.parse_args()


def workload_desc(inst):
    p = inst.params
    return (f"{inst.name}: 3-deep loop stencil MAP, blockDim {inst.n_threads}, T={p['T']} phases, "
            f"R={p['R']} rows/thread, C={p['C']} cols, ping-pong (DRF)") if inst.name[0] == "5" else inst.name


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    PERIOD_MS = 50

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"mapcheck_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", str(self.PERIOD_MS)], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # the timed region is short (tens of ms per step): wait for the first sample
        t0 = time.time()
        while time.time() - t0 < 5.0:
            try:
                if os.path.getsize(self.path) > 0:
                    break
            except OSError:
                pass
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(2.5 * self.PERIOD_MS / 1e3)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
                except ValueError:
                    continue
        if not rows:
            return None
        mx = max(r[1] for r in rows)
        loaded = [r for r in rows if r[0] > 0.5 * mx] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------- CPU oracle -----
def oracle_sample(inst_full, rows):
    """Bounded sample of the same workload: phase 0 only (T=1), `rows` rows per thread."""
    name = inst_full.name
    if name[0] == "5":
        p = inst_full.params
        return config(name, block=inst_full.n_threads, T=1, R=rows, C=p["C"])
    return inst_full


def run_oracle(inst, threads):
    import oracle
    t0 = time.perf_counter()
    r = oracle.check_instance(inst, threads=threads)
    dt = time.perf_counter() - t0
    if r.status != 0:
        raise RuntimeError(f"oracle failed: {r.diag}")
    return r, dt


def sample_text(inst):
    p = inst.params
    return (f"{inst.name} with T={p.get('T')}, R={p.get('R')} (phase 0, rows 0..R-1 of every thread): "
            f"{inst.n_threads}x{p.get('R')}x{p.get('C')}x4 accesses")


def reference_arm(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on the host cores."""
    if rank != 0:
        return
    inst = config(args.config)
    samp = oracle_sample(inst, args.ref_rows)
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        run_oracle(samp, cores)
    times, n = [], 0
    for _ in range(args.steps):
        r, dt = run_oracle(samp, cores)
        times.append(dt)
        n = r.n_accesses
    tot = sum(times)
    value = n * len(times) / tot / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "ranks": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "config": {"workload": workload_desc(inst), "sample": sample_text(samp)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample_text(samp)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours ----
def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(which):
    """dram bytes per launch of a kernel from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", f"ncu_{which}_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


# Roofline models of the kernels that can dominate a step (all HBM-bound; the
# library reports their algorithmic bytes per launch).
ROOFLINE_MODELS = {
    "direct": ("generate fused with the direct-address table reductions (gen_0, mode direct)", "direct",
               "2 x table bytes per launch: every cell of the 2^S-cell table read and written once "
               "(the reductions are served by L2; row-jammed, 0.133 red.or.b64 per 5a access, see red); "
               "bound by the L2's rate of atomic updates into the HBM-resident table "
               "(profiles/r1h_red_width_microbench.txt); the issue view is under alu. "
               "Over compressible scratch (config.scratch) the zero-filled lines the reductions fill "
               "compress, so the measured DRAM traffic (traffic) is below these algorithmic bytes"),
    "onesweep": ("k_rsweep (static-range LSD radix pass)", "rsweep", "16 B per key per active pass (8 read + 8 write)"),
}


# Issue peak of a B200 (B200_PROFILING.md / B300_MICROARCH.md unit counts): 148 SMs x
# 4 schedulers x 1 warp-instruction per cycle x 1965 MHz = 1163 G warp-instructions/s.
ISSUE_PEAK_G = 148 * 4 * 1.965


def ncu_direct():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_direct_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# Global red.or.b64 ceiling into a 2 GiB (HBM-resident) table, measured on this pool's
# B200s: 4.03 TB/s of 8-byte payload (profiles/r1h_red_width_microbench.txt).
RED64_CEILING_TBS = 4.03


def issue_roofline(kern, hbm, acc_per_launch=None, reds_per_access=0.25):
    """The direct generate: primary view HBM (2 x table bytes per launch over its live
    CUDA-event time; DRAM traffic = algorithmic in the committed ncu capture).  Since the
    r1t/r1u instruction cuts it is no longer issue-bound (issue ~61% alone, r1w): what
    limits it is the rate of global red.or.b64 into an HBM-resident table
    (profiles/r1h_red_width_microbench.txt).  The issue view -- warp instructions per
    launch from the same capture over the live duration, against the derived issue
    peak -- is kept under "alu"."""
    info = ncu_direct()
    inst = info.get("warp_inst_per_launch")
    k = kern.get("direct", {})
    if not inst or not k.get("launches") or k.get("ms", 0) <= 0:
        return hbm
    per_launch_s = k["ms"] / 1e3 / k["launches"]
    achieved = inst / per_launch_s / 1e9
    out = dict(hbm)
    if acc_per_launch:
        # 16-bit cells in aligned quads: one red.or.b64 per 4 accesses (5a: every site
        # unit-stride, every quad aligned); row-jammed by JU rows per thread, a row's
        # three reads fold into one reduction: (JU + 2 + JU) per 16 JU accesses
        red_tbs = acc_per_launch * reds_per_access * 8 / per_launch_s / 1e12
        out["red"] = {"achieved": red_tbs, "peak": RED64_CEILING_TBS, "unit": "TB/s of red.or.b64 payload",
                      "peak_kind": "measured microbenchmark (profiles/r1h_red_width_microbench.txt)",
                      "frac": red_tbs / RED64_CEILING_TBS,
                      "reds_per_access": reds_per_access,
                      "work_model": f"accesses x {reds_per_access:.4f} red.or.b64 of 8 B per launch"}
    out["alu"] = {"achieved": achieved, "peak": ISSUE_PEAK_G,
                  "peak_kind": "derived: 148 SMs x 4 schedulers x 1.965 GHz (one warp-instruction per scheduler-cycle)",
                  "unit": "G warp-inst/s", "frac": achieved / ISSUE_PEAK_G,
                  "work_model": f"{inst:.4g} warp instructions per launch (ncu smsp__inst_executed of the bench "
                                f"command, issue active {info.get('issue_active_pct', float('nan')):.0f}% when alone)"}
    return out


def kernel_roofline(kern, cls, peak, peak_kind):
    """achieved = the class's algorithmic bytes / its CUDA-event time; for the radix
    pass both launch forms (plain, and building the next pass's range table) together."""
    z = {"ms": 0, "bytes": 0, "launches": 0}
    parts = None
    if cls == "onesweep":
        a, b = kern.get("onesweep", z), kern.get("onesweep_next", z)
        k = {f: a[f] + b[f] for f in ("ms", "bytes", "launches")}
        gbs = lambda d: (d["bytes"] / (d["ms"] / 1e3) / 1e9) if d["ms"] > 0 else None
        parts = {"plain_pass_GB_s": gbs(a), "next_table_pass_GB_s": gbs(b), "plain_launches": a["launches"],
                 "next_table_launches": b["launches"]}
    else:
        k = kern.get(cls, z)
    achieved = (k["bytes"] / (k["ms"] / 1e3) / 1e9) if k["ms"] > 0 else 0.0
    name, tag, model = ROOFLINE_MODELS[cls]
    out = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
           "unit": "GB/s", "frac": achieved / peak if peak else None, "traffic": ncu_traffic(tag),
           "bytes_model": model, "launches": k["launches"]}
    if parts:
        out["parts"] = parts
    return out


def kernel_table(results):
    """Per-class totals over the results.  With sampled timing (profile="sampled") only
    some launches carry events: "ms" is then the timed launches' average duration times
    every launch of the class (the estimate of the class's total), "timed" how many
    launches were actually timed."""
    kern = {}
    for r in results:
        for k, v in (r.kernels or {}).items():
            d = kern.setdefault(k, {"ms_timed": 0.0, "launches": 0, "bytes": 0, "timed": 0})
            d["ms_timed"] += v["ms"]
            d["launches"] += v["launches"]
            d["bytes"] += v["bytes"]
            d["timed"] += v.get("timed", v["launches"])
    for d in kern.values():
        d["ms"] = d["ms_timed"] / d["timed"] * d["launches"] if d["timed"] else 0.0
    return kern


def _free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def relaunch(n):
    """--gpus N > 1 without a torchrun environment: run this script as N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
        reference_arm(args, rank, world)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    import torch
    import torch.distributed as dist
    import paper_2203_12878_b200 as mc
    from paper_2203_12878_b200.dist import reduce_results

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    inst = config(args.config)
    prog = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
    names = prog.array_names()
    if not args.chunk:
        args.chunk = prog.default_chunk(world)
    # scratch (key buffers / direct tables) from the library's allocator helper:
    # compressible device memory when the driver grants it (the tables are cleared
    # to zero before every chunk; zero lines compress -- include/mapcheck.h
    # map_scratch_alloc), plain device memory with --plain-scratch
    if args.plain_scratch:
        scratch = torch.empty(prog.scratch_bytes(args.chunk), dtype=torch.uint8, device="cuda")
        scratch_kind = "plain device memory (torch.empty)"
    else:
        scratch = mc.alloc_scratch(prog.scratch_bytes(args.chunk))
        scratch_kind = ("compressible device memory (map_scratch_alloc, generic compression granted)"
                        if scratch._map_block.compressed else "plain device memory (map_scratch_alloc: "
                        "compression not granted)")
    stream = torch.cuda.current_stream()
    n_chunks = prog.n_chunks(args.chunk)
    my_chunks = prog.rank_chunks(rank, world, args.chunk)

    def step(profile=False, detect=args.detect):
        if args.mode == "exchange" and world > 1:
            from paper_2203_12878_b200.dist import check_races_exchange
            return check_races_exchange(prog, scratch, stream, args.chunk)
        r = prog.check_races(scratch=scratch, stream=stream, chunk_max_accesses=args.chunk, rank=rank,
                             world=world, profile=profile, detect=detect)
        if world > 1:
            r = reduce_results(r, names, device=torch.device("cuda", local))
        return r

    # warm-up with the timed steps' own flags: the library captures the second
    # identical call into a CUDA graph (per-launch timing events included, as
    # event-record nodes) and the timed steps replay it
    for _ in range(max(args.warmup, 0)):
        step(profile="sampled")

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    results = []
    for _ in range(args.steps):
        # CUDA events around the generate launches of every fourth chunk only
        # (MAP_EXEC_PROFILE_GENERATE | MAP_EXEC_PROFILE_SAMPLED, 4 of 5a's 16 per step;
        # profiles/r2zq_prof_overhead.json: events on all 16 cost 1.6% of the step):
        # the roofline's kernel is timed live inside the timed region; the other
        # classes are counted here and timed in two extra steps after it
        results.append(step(profile="sampled"))
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_acc = sum(r.n_accesses for r in results)          # already summed over ranks
    value = total_acc / (ms_max / 1e3) / 1e9

    # per-kernel-class device time (this rank) over the timed steps: the generate
    # classes from the timed steps themselves; the breakdown of the other classes
    # from two fully profiled steps after the timed region (scaled to the same
    # step count), so the shares and pipeline bytes describe the same run
    kern = kernel_table(results)
    full = [step(profile=True) for _ in range(2)][1:]
    k_full = kernel_table(full)
    for cls, v in k_full.items():
        if kern.get(cls, {}).get("ms", 0) == 0 and v["ms"] > 0:
            kern[cls] = dict(kern.get(cls, v))
            kern[cls]["ms"] = v["ms"] * len(results) / len(full)
            kern[cls]["timed_after"] = True
    launches = sum(r.gpu_launches for r in results)
    peak, peak_kind = measured_peak()
    # the dominant kernel of the path that ran: the fused direct generate, or the radix pass
    ms_of = lambda c: kern.get(c, {}).get("ms", 0) + (kern.get("onesweep_next", {}).get("ms", 0) if c == "onesweep" else 0)
    dominant = max(ROOFLINE_MODELS, key=ms_of)
    roofline = kernel_roofline(kern, dominant, peak, peak_kind)
    # reductions per access of the direct generate: 5a's stencil (three reads of a row,
    # one write) in quads, row-jammed by JU rows per thread when the JIT took the jam
    import re as _re
    _m = _re.search(r"u_ < (\d+)u", prog.jit_source(0, 1)) if inst.name[0] == "5" else None
    ju = int(_m.group(1)) if _m else 0
    reds_per_access = (2 * ju + 2) / (16 * ju) if ju else 0.25
    if dominant == "direct":
        acc_launch = sum(r.n_accesses for r in results) / max(1, kern.get("direct", {}).get("launches", 0))
        roofline = issue_roofline(kern, roofline, acc_launch, reds_per_access)
    kern_total = sum(v["ms"] for v in kern.values()) or 1.0
    pipe_bytes = sum(v["bytes"] for v in kern.values())
    # the dominant kernel alone: the direct path's chunks run one after another
    # (MAP_EXEC_SEQUENTIAL), so its CUDA-event time is not shared with the
    # overlapped scans (reported next to the live, overlapped figure)
    if dominant == "direct" and kern.get("direct", {}).get("launches"):
        solo = [prog.check_races(scratch=scratch, stream=stream, chunk_max_accesses=args.chunk, rank=rank,
                                 world=world, profile=True, detect=args.detect, overlap=False) for _ in range(2)]
        k_solo = kernel_table(solo[1:])
        r_solo = issue_roofline(k_solo, kernel_roofline(k_solo, "direct", peak, peak_kind),
                                solo[1].n_accesses / max(1, k_solo.get("direct", {}).get("launches", 0)),
                                reds_per_access)
        roofline["solo"] = {"achieved": r_solo["achieved"], "frac": r_solo["frac"], "unit": r_solo["unit"],
                            "red_frac": r_solo.get("red", {}).get("frac"),
                            "note": "same kernel, chunks run sequentially (no concurrent scans)"}
    kernels_out = {k: {"ms_per_step": v["ms"] / len(results), "share": v["ms"] / kern_total,
                       "GB_s": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 and v["bytes"] else None,
                       "launches_per_step": v["launches"] / len(results),
                       "timed": "after the timed region (2 profiled steps)" if v.get("timed_after") else
                                f"live, inside the timed region ({v['timed']} of {v['launches']} launches "
                                f"carried events)"} for k, v in kern.items()}

    # e2e: the public API from host text to host verdict, every step (compile + H2D bytecode + D2H result)
    e2e = None
    if not args.no_e2e:
        # warm-up of the end-to-end leg itself (first-use costs of a fresh program in
        # this process: pinned staging buffer, side streams, events -- pooled after)
        for _ in range(max(args.warmup, 1)):
            p2 = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
            p2.check_races(scratch=scratch, stream=stream, chunk_max_accesses=args.chunk, rank=rank, world=world,
                           detect=args.detect)
            del p2
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_res = []
        for _ in range(args.steps):
            p2 = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
            r = p2.check_races(scratch=scratch, stream=stream, chunk_max_accesses=args.chunk, rank=rank, world=world,
                               detect=args.detect)
            if world > 1:
                r = reduce_results(r, names, device=torch.device("cuda", local))
            e_res.append(r)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        w = torch.tensor([wall], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(w, op=dist.ReduceOp.MAX)
        wall = float(w.item())
        e2e = {"value": sum(r.n_accesses for r in e_res) / wall / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": results[0].h2d_bytes, "d2h_bytes_per_step": results[0].d2h_bytes,
               "includes": "map_compile from MAP text + map_check_races (bytecode/segment H2D, result D2H)"}

    # the other detect paths on the same workload, for context (same timing rules):
    # the bucket-table path and the full sort (the north_star's generate -> sort -> detect)
    alt, roof_sort = None, None
    if not args.no_alt_path:
        alt = {"identical_result": True, "scratch": "plain device memory (torch.empty): the keys paths scatter "
                                                    "incompressible keys, slower in compressible memory"}
        if not args.plain_scratch:
            del scratch
            torch.cuda.synchronize()
            scratch = torch.empty(prog.scratch_bytes(args.chunk), dtype=torch.uint8, device="cuda")
        for alt_mode in [m for m in ("table", "sort") if m != args.detect]:
            step(detect=alt_mode)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            a_res = [step(profile=True, detect=alt_mode) for _ in range(args.steps)]
            a1.record(stream)
            torch.cuda.synchronize()
            ta = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(ta, op=dist.ReduceOp.MAX)
            same = all((x.verdict, x.witness, x.n_accesses, x.racy_segments) ==
                       (results[0].verdict, results[0].witness, results[0].n_accesses, results[0].racy_segments)
                       for x in a_res)
            alt[alt_mode] = sum(x.n_accesses for x in a_res) / (float(ta.item()) / 1e3) / 1e9
            alt["identical_result"] = alt["identical_result"] and same
            if alt_mode == "table":
                k_alt = kernel_table(a_res)
                roof_sort = kernel_roofline(k_alt, "onesweep", peak, peak_kind)
                roof_sort["path"] = "table (partial LSD sort + bucket tables)"

    # the other config families at full size (context for the same metric; the
    # library's automatic path, CUDA-graph replays, best of 3 device times)
    others = None
    if not args.no_other_configs and world == 1 and args.mode == "shard":
        others = {}
        for name in ("3a", "3b", "4a", "4b", "4c", "4d", "2b", "1a"):
            oi = config(name)
            op = mc.MapProgram(oi.src, oi.grid, oi.block, oi.params)
            osc = (torch.empty(op.scratch_bytes(), dtype=torch.uint8, device="cuda") if args.plain_scratch
                   else mc.alloc_scratch(op.scratch_bytes()))
            for _ in range(2):
                orr = op.check_races(scratch=osc, stream=stream)
            ms_o = min(op.check_races(scratch=osc, stream=stream).device_ms for _ in range(3))
            prof = op.check_races(scratch=osc, stream=stream, profile=True).kernels
            path = max((v["ms"], k) for k, v in prof.items() if k in ("unit", "direct", "onesweep", "detect"))[1]
            others[name] = {"G_acc_s": orr.n_accesses / ms_o / 1e6, "ms": ms_o, "n_accesses": orr.n_accesses,
                            "verdict": "racy" if orr.verdict else "drf", "main_kernel": path}
            del osc

    # NEXT-2 context: a data-carrying BabyCUDA transpose at config-3 scale (2^16 blocks
    # x 256 threads) executed on the GPU (Fig. 5 semantics) and its executed access set
    # checked against the inferred MAP's (Theorem 1)
    next2 = None
    if not args.no_other_configs and world == 1 and args.mode == "shard":
        from workloads import babycuda as wb
        ki = wb.kernel("transpose", ts=32, rw=8, grid=65536)
        kern = mc.Kernel(ki.src, ki.grid, ki.block, ki.params)
        kern.execute()
        ex_ms = min(kern.execute().device_ms for _ in range(3))
        kr = kern.execute()
        diff = kern.theorem1_diff(mc.MapProgram(mc.infer(ki.src).map_text, ki.grid, ki.block, ki.params))
        next2 = {"kernel": "BabyCUDA tiled transpose 32x32, 2^16 blocks x 256 threads (workloads/babycuda.py)",
                 "executed_accesses": kr.n_events, "exec_ms": ex_ms, "G_events_s": kr.n_events / ex_ms / 1e6,
                 "typable": kr.typable, "theorem1_equal": diff.equal, "access_values": diff.n_alpha,
                 "verdict": "racy" if kr.verdict else "drf"}

    cpu = None
    if world > 1:
        dist.barrier()          # the GPU timing is done on every rank before the CPU leg
    if rank == 0 and not args.no_cpu_baseline:
        samp = oracle_sample(inst, args.cpu_rows)
        cores = os.cpu_count() or 1
        orc, dt = run_oracle(samp, cores)
        cpu = {"value": orc.n_accesses / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": sample_text(samp), "seconds": dt}

    if rank == 0:
        r0 = results[-1]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / len(results), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": workload_desc(inst), "n_accesses": r0.n_accesses, "chunks": n_chunks,
                       "chunk_max_accesses": args.chunk, "rank0_chunks": len(my_chunks),
                       "parallelism": (f"dp{world}: each rank a contiguous bound-balanced range of chunks, no "
                                       f"data-path collective" if args.mode == "shard" else
                                       f"key exchange over {world} ranks (all_to_all_single)"),
                       "l2": "inputs larger than L2: a 1 GiB direct-address table of 16-bit cells (or 8 GiB of "
                             "keys) per chunk vs 126 MB L2; no flush needed",
                       "scratch": scratch_kind,
                       "verdict": "racy" if r0.verdict else "drf",
                       "witness": list(r0.witness.as_tuple()) if r0.witness else None},
            "roofline": roofline,
            "roofline_sort_path": roof_sort,
            "kernels": kernels_out,
            "detect_path": args.detect if args.detect != "auto" else "auto (direct-address table for dense chunks)",
            "detect_paths": alt,
            "pipeline_bytes_per_access": pipe_bytes / max(1, total_acc),
            "pipeline_hbm": {"achieved": pipe_bytes / (ms_max / 1e3) / 1e9, "peak": peak,
                             "frac": pipe_bytes / (ms_max / 1e3) / 1e9 / peak if peak else None,
                             "note": "algorithmic bytes of every kernel of the timed steps / the steps' device time "
                                     "(the direct pipeline overlaps the table scans with the next generate); over "
                                     "compressible scratch (config.scratch) the cleared tables' zero lines compress, "
                                     "so the physical DRAM traffic is lower than these bytes and frac can exceed 1 "
                                     "(profiles/*_direct_ncu_full.txt: the generate's DRAM traffic per launch)"},
            "other_configs": others,
            "babycuda_executor": next2,
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
