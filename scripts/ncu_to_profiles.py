"""Write the ncu evidence bench.py and DESIGN.md cite into profiles/.

usage: python scripts/ncu_to_profiles.py <full .ncu-rep> <launch-list .csv> <tag>
  profiles/<tag>_ncu_full.txt       per-kernel summary of the --set full capture
  profiles/<tag>_launches.csv       the launch list (gpu__time_duration per launch)
  profiles/<tag>_launch_shares.txt  device time per kernel class from the launch list
  profiles/ncu_rsweep_traffic.json  dram bytes per launch of the radix pass (bench.py roofline.traffic)
"""
import csv, io, json, os, re, shutil, subprocess, sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main(rep, launches, tag):
    prof = os.path.join(ROOT, "profiles")
    hdr, units, rows = raw_rows(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    lines, traffic, direct = [], None, None
    for r in rows:
        name = r[idx["Kernel Name"]]
        get = lambda k: float(r[idx[k]]) if k in idx and r[idx[k]] else float("nan")
        dur_unit = units[idx["gpu__time_duration.sum"]]
        dur = get("gpu__time_duration.sum") * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(dur_unit, 1e-9)
        bu = units[idx["dram__bytes_read.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu, 1)
        rd, wr = get("dram__bytes_read.sum") * scale, get("dram__bytes_write.sum") * scale
        lines.append(f"{name.split('(')[0]:40s} dur {dur*1e3:8.3f} ms  dram read {rd/1e9:7.3f} GB  write {wr/1e9:7.3f} GB  "
                     f"-> {(rd+wr)/dur/1e9:7.1f} GB/s  issue {get('smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f}%  "
                     f"occupancy {get('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}%  regs {get('launch__registers_per_thread'):.0f}")
        if name.startswith("gen_") and (direct is None or dur > direct["duration_s"]):
            # the direct-mode generate (the longest gen_ launch: the filter pass exits at once when DRF)
            direct = {"kernel": name.split("(")[0] + " (mode direct)", "dram_bytes_per_launch": rd + wr, "dram_read": rd,
                      "dram_write": wr, "duration_s": dur, "source": os.path.basename(rep),
                      "warp_inst_per_launch": get("smsp__inst_executed.sum"),
                      "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active")}
        if "k_rsweep" in name and traffic is None:
            traffic = {"kernel": name.split("(")[0], "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                       "duration_s": dur, "source": os.path.basename(rep)}
    with open(os.path.join(prof, f"{tag}_ncu_full.txt"), "w") as f:
        f.write("# ncu --set full --clock-control none (one launch per kernel; replayed, cold-cache)\n")
        f.write("\n".join(lines) + "\n")
    if traffic:
        with open(os.path.join(prof, "ncu_rsweep_traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    if direct and "direct" in tag:
        with open(os.path.join(prof, "ncu_direct_traffic.json"), "w") as f:
            json.dump(direct, f, indent=1)
    # launch list -> shares
    shutil.copy(launches, os.path.join(prof, f"{tag}_launches.csv"))
    txt = open(launches).read()
    start = txt.find('"ID"')
    agg = defaultdict(lambda: [0.0, 0])
    for r in csv.DictReader(io.StringIO(txt[start:])):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
        k = re.sub(r"<.*>", "", k)
        v = float(r["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1, "msecond": 1}.get(r["Metric Unit"], 1e-6)
        agg[k][0] += v
        agg[k][1] += 1
    tot = sum(v[0] for v in agg.values())
    with open(os.path.join(prof, f"{tag}_launch_shares.txt"), "w") as f:
        f.write(f"# device time per kernel from {os.path.basename(launches)} (ncu launch list, serialised, cold-cache)\n")
        for k, (ms, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
            f.write(f"{k:40s} {ms:10.3f} ms  {100*ms/tot:5.1f}%  launches {n}\n")
        f.write(f"{'total':40s} {tot:10.3f} ms\n")


if __name__ == "__main__":
    main(*sys.argv[1:4])
