"""Summaries of ncu captures for profiles/ (run here, on the .ncu-rep / .csv
that gpurun brought back).

    python tools/profile_summary.py report  gpurun_out/prof_level.ncu-rep  > profiles/rNN_ncu_level.txt
    python tools/profile_summary.py launches gpurun_out/launches.csv       > profiles/rNN_launches.txt
    python tools/profile_summary.py traffic gpurun_out/prof_query.ncu-rep  > profiles/ncu_traffic.json

`report`: per kernel the SOL / occupancy / memory figures and the SURVEY 8(d)
counters (dram bytes, L2 hit rate, sectors, warps active).  `launches`: the
launch list of one bench command grouped by kernel with each kernel's share of
device time (cold-cache, serialised: shares, not absolutes).  `traffic`: dram
bytes per query of the query kernels, read by bench.py's roofline.traffic.
"""

import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict

DETAILS = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
           "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
           "Achieved Occupancy", "Theoretical Occupancy", "L2 Hit Rate", "L1/TEX Hit Rate",
           "Mem Busy", "Max Bandwidth", "Executed Instructions", "Grid Size", "Block Size",
           "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction",
           "Eligible Warps Per Scheduler")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
       "lts__t_sectors_op_read.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
       "sm__warps_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
       "launch__registers_per_thread")
STALLS = re.compile(r"^smsp__pcsamp_warps_issue_stalled_([a-z_]+)$")


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_rows(rep):
    rows = ncu_csv(rep, "raw")
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def report(rep):
    rows = ncu_csv(rep, "details")
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    det = OrderedDict()
    for r in rows[1:]:
        key = (r[ix["ID"]], r[ix["Kernel Name"]])
        if r[ix["Metric Name"]] in DETAILS:
            det.setdefault(key, []).append((r[ix["Metric Name"]], r[ix["Metric Value"]],
                                            r[ix["Metric Unit"]]))
    hdr, units, data = raw_rows(rep)
    for n, ((kid, name), vals) in enumerate(det.items()):
        print(f"=== [{kid}] {name}")
        for k, v, u in vals:
            print(f"  {k:42s} {v:>16s} {u}")
        if n < len(data):
            d = dict(zip(hdr, data[n]))
            un = dict(zip(hdr, units))
            for k in RAW:
                if k in d:
                    print(f"  {k:60s} {d[k]:>16s} {un.get(k, '')}")
            st = sorted(((int(float(d[k] or 0)), STALLS.match(k).group(1)) for k in d
                         if STALLS.match(k) and "not_issued" not in k), reverse=True)
            tot = sum(s for s, _ in st) or 1
            print("  stall samples: " + ", ".join(f"{nm} {100 * s / tot:.1f}%"
                                                  for s, nm in st[:8] if s))
        print()


def launches(path):
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = OrderedDict()
    for r in rows[1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ix["Kernel Name"]])
        unit = r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    total = sum(a[1] for a in agg.values()) or 1
    print(f"{'kernel':60s} {'launches':>8s} {'total us':>12s} {'share':>7s}")
    for name, (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:60]:60s} {c:8d} {us:12.1f} {100 * us / total:6.1f}%")
    print(f"{'TOTAL':60s} {sum(a[0] for a in agg.values()):8d} {total:12.1f}")


def traffic(rep, queries_per_launch):
    hdr, units, data = raw_rows(rep)
    un = dict(zip(hdr, units))
    out = {}
    for r in data:
        d = dict(zip(hdr, r))
        m = re.match(r"void (\w+)", d["Kernel Name"])
        if not m:
            continue
        b = (to_bytes(d["dram__bytes_read.sum"], un["dram__bytes_read.sum"]) +
             to_bytes(d["dram__bytes_write.sum"], un["dram__bytes_write.sum"]))
        out[m.group(1)] = {"dram_bytes": b, "queries": queries_per_launch,
                           "dram_bytes_per_query": b / queries_per_launch}
    print(json.dumps(out, indent=1))


def traffic_csv(path, queries_per_launch):
    """dram bytes per query from a `--metrics dram__bytes_*` launch CSV taken
    at the bench's own batch size (one launch per kernel)."""
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    acc = {}
    for r in rows[1:]:
        m = re.match(r"void (\w+)", r[ix["Kernel Name"]]) or re.match(r"(\w+)", r[ix["Kernel Name"]])
        name = m.group(1).split("::")[-1]
        metric = r[ix["Metric Name"]]
        if metric.startswith("dram__bytes"):
            acc.setdefault(name, 0.0)
            acc[name] += to_bytes(r[ix["Metric Value"]], r[ix["Metric Unit"]])
    out = {k: {"dram_bytes": v, "queries": queries_per_launch,
               "dram_bytes_per_query": v / queries_per_launch} for k, v in acc.items()}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    cmd, path = sys.argv[1], sys.argv[2]
    if cmd == "report":
        report(path)
    elif cmd == "launches":
        launches(path)
    elif cmd == "traffic":
        traffic(path, int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000)
    elif cmd == "traffic_csv":
        traffic_csv(path, int(sys.argv[3]) if len(sys.argv) > 3 else 33_333_334)
    else:
        raise SystemExit(__doc__)
