"""One table for every kernel of an `ncu --set full` raw-page CSV
(scripts/gpu_ncu_all.sh -> gpurun_out/prof_all_raw.csv):

    python tools/ncu_all_summary.py gpurun_out/prof_all_raw.csv [peak_GBps] > profiles/r02_ncu_all_kernels.txt

Per kernel (the launch with the most DRAM bytes of each name -- the
representative full-size launch): duration, DRAM bytes read + written,
achieved DRAM GB/s and its fraction of the measured HBM peak, ncu's own
dram__throughput %, L2 hit rate, achieved occupancy, registers, IPC, and
the top warp-stall reasons (pc sampling).
"""

import csv
import io
import json
import os
import re
import sys

STALL = re.compile(r"^smsp__pcsamp_warps_issue_stalled_([a-z_]+)$")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
         "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}


def num(v, unit=""):
    try:
        x = float(str(v).replace(",", ""))
    except ValueError:
        return 0.0
    return x * SCALE.get(unit, 1.0)


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    return name.replace("<unnamed>::", "").replace("wt::", "").replace("unsigned char", "u8").replace(
        "unsigned short", "u16").replace("unsigned long long", "u64")


def main(path, peak):
    with open(path) as f:
        rows = list(csv.reader(io.StringIO("".join(l for l in f if not l.startswith("==")))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    un = dict(zip(hdr, units))
    best = {}
    counts = {}
    for r in data:
        d = dict(zip(hdr, r))
        k = short(d.get("Kernel Name", "?"))
        if not k.startswith(("wlevel", "wlast", "qlayout", "hist", "block_l1", "l1_scan",
                             "wcount0", "first_outside", "bits_", "access_kernel", "rank_kernel",
                             "select_kernel", "qsort", "qunsort", "map_kernel", "encode_kernel",
                             "split_", "pack_bits", "wpair", "dir_kernel", "dirq_kernel", "widen")):
            continue
        counts[k] = counts.get(k, 0) + 1
        b = (num(d.get("dram__bytes_read.sum", 0), un.get("dram__bytes_read.sum", "")) +
             num(d.get("dram__bytes_write.sum", 0), un.get("dram__bytes_write.sum", "")))
        if k not in best or b > best[k][0]:
            best[k] = (b, d)
    print(f"# every kernel of libwt_b200.so, one representative (largest-DRAM) launch each;"
          f" peak {peak:.1f} GB/s (MEASURED_PEAKS.json hbm_gbs)")
    print(f"{'kernel':46s} {'n':>3s} {'us':>9s} {'DRAM MB':>9s} {'GB/s':>8s} {'frac':>5s} "
          f"{'dram%':>6s} {'L2hit':>6s} {'occ%':>5s} {'regs':>4s} {'IPC':>5s}  top stalls")
    out = {}
    for k, (b, d) in sorted(best.items(), key=lambda kv: -kv[1][0]):
        us = num(d.get("gpu__time_duration.sum", 0), un.get("gpu__time_duration.sum", ""))
        gbs = b / (us * 1e-6) / 1e9 if us else 0.0
        st = sorted(((num(d[c]), STALL.match(c).group(1)) for c in d
                     if STALL.match(c) and "not_issued" not in c), reverse=True)
        tot = sum(s for s, _ in st) or 1.0
        stalls = ", ".join(f"{nm} {100 * s / tot:.0f}%" for s, nm in st[:3] if s)
        rec = {
            "launches": counts[k], "us": us, "dram_bytes": b, "GB_per_s": gbs,
            "frac_of_hbm": gbs / peak,
            "dram_pct": num(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0)),
            "l2_hit_pct": num(d.get("lts__t_sector_hit_rate.pct", 0)),
            "occupancy_pct": num(d.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0)),
            "regs": num(d.get("launch__registers_per_thread", 0)),
            "ipc": num(d.get("sm__inst_executed.avg.per_cycle_active", 0)),
            "stalls": stalls}
        out[k] = rec
        print(f"{k[:46]:46s} {counts[k]:3d} {us:9.1f} {b / 1e6:9.1f} {gbs:8.1f} "
              f"{rec['frac_of_hbm']:5.2f} {rec['dram_pct']:6.1f} {rec['l2_hit_pct']:6.1f} "
              f"{rec['occupancy_pct']:5.1f} {rec['regs']:4.0f} {rec['ipc']:5.2f}  {stalls}")
    if len(sys.argv) > 3:
        with open(sys.argv[3], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    peak = float(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else json.load(
        open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "MEASURED_PEAKS.json")))["hbm_gbs"]
    main(sys.argv[1], peak)
