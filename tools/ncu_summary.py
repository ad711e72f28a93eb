"""Summarise ncu artifacts (launch-list CSV, --set full reports) into tracked text files.

    python tools/ncu_summary.py launches <csv> > profiles/<name>.txt
    python tools/ncu_summary.py report <ncu-rep> > profiles/<name>.txt
"""
import collections
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread",
        "Achieved Occupancy", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "sm__inst_executed_pipe_tensor_op_dmma.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        key = (r[0], r[ki])
        per.setdefault(key, {})[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.OrderedDict()
    for (_, name), m in per.items():
        short = name.split("(")[0][:70]
        a = agg.setdefault(short, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list: {path}  ({len(per)} launches, cold-cache serialised; compare SHARES)")
    print(f"{'kernel':72s} {'n':>5s} {'time_us':>11s} {'share':>7s} {'dram_MB':>9s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:72s} {n:5d} {t / 1e3:11.1f} {100 * t / tot:6.1f}% {b / 1e6:9.1f}")


def report(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(det.splitlines()))
    hdr = rows[0]
    ii, ki, mi, vi, ui = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    by = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] in KEYS:
            by.setdefault((r[ii], r[ki][:90]), {})[r[mi]] = f"{r[vi]} {r[ui]}"
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    rh = rr[0]
    units = dict(zip(rh, rr[1])) if len(rr) > 1 else {}
    rawvals = [dict(zip(rh, r)) for r in rr[2:]]
    print(f"# ncu --set full: {path}")
    for n, ((i, k), m) in enumerate(by.items()):
        print(f"\n## launch {i}: {k}")
        for key in KEYS:
            if key in m:
                print(f"  {key:40s} {m[key]}")
        if n < len(rawvals):
            for key in RAW:
                if key in rawvals[n]:
                    print(f"  {key:40s} {rawvals[n][key]} {units.get(key, '')}".rstrip())


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
