"""Summarise an .ncu-rep: per kernel launch, the metrics that decide the roofline."""
import csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "dur_ns"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__inst_executed.sum", "inst"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "inst_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "st_lsb"),
]


def main(path, kfilter=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        if kfilter not in name:
            continue
        vals = []
        for k, short in KEYS:
            if k in idx:
                vals.append(f"{short}={r[idx[k]]}")
        stalls = sorted(((h, r[i]) for h, i in idx.items() if h.startswith("smsp__average_warps_issue_stalled_")
                         and h.endswith("_per_issue_active.ratio")), key=lambda x: -float(x[1] or 0))[:5]
        print(name.split("(")[0], " ".join(vals))
        print("   stalls/issue:", ", ".join(f"{h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={v}" for h, v in stalls))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
