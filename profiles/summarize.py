"""Summaries of ncu outputs committed under profiles/ (run here, no GPU).

    python profiles/summarize.py launches <launches.csv>   # per-kernel share of a launch list
    python profiles/summarize.py rep <report.ncu-rep>      # key metrics of a --set full capture
"""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total us':>12s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:70]:70s} {c:8d} {t:12.1f} {100 * t / tot:5.1f}%")
    print(f"total {tot / 1e3:.2f} ms over {sum(c for c, _ in agg.values())} launches "
          "(cold-cache, serialised by ncu: compare shares, not absolutes)")


KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Registers Per Thread", "Grid Size",
        "Block Size", "Theoretical Occupancy", "Achieved Occupancy", "Issue Slots Busy",
        "Executed Ipc Active", "SM Busy", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "No Eligible",
        "Executed Instructions"]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = csv.reader(out.splitlines())
    h = next(r)
    kn = h.index("Kernel Name")
    for row in r:
        name, unit, val = row[-3], row[-2], row[-1]
        if any(name.startswith(k) for k in KEYS) or name.startswith("INF") or row[-4] in ("INF",):
            print(f"{row[kn][:40]:40s} | {name[:60]:60s} | {unit:8s} | {val}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    hdr = next(csv.reader([raw[0]]))
    vals = list(csv.reader(raw[2:]))
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64",
            "sm__pipe_fp64_cycles_active", "smsp__inst_executed.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed_pipe_fp64.sum", "gpu__time_duration.sum"]
    for v in vals:
        for i, c in enumerate(hdr):
            if any(c.startswith(w) for w in want):
                print(f"raw | {c:70s} | {v[i]}")


if __name__ == "__main__":
    {"launches": launches, "rep": rep}[sys.argv[1]](sys.argv[2])
