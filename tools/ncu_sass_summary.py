"""Summarise an ncu report's SASS page: stall samples and executed
instructions per opcode, plus the hottest instructions.

    python tools/ncu_sass_summary.py report.ncu-rep [kernel-regex]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def main():
    rep = sys.argv[1]
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if len(sys.argv) > 2:
        cmd += ["-k", "regex:" + sys.argv[2]]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    blocks = re.split(r'^"Kernel Name",', out, flags=re.M)
    for blk in blocks[1:]:
        name, rest = blk.split("\n", 1)
        rows = list(csv.reader(io.StringIO(rest)))
        hdr, rows = rows[0], rows[1:]
        ix = {h: i for i, h in enumerate(hdr)}
        by_op = collections.Counter()
        stall = collections.Counter()
        tot_i = tot_s = 0
        hot = []
        for r in rows:
            if len(r) < len(hdr):
                continue
            src = r[ix["Source"]].strip()
            op = src.split()[0] if src else "?"
            if op.startswith("@"):
                op = src.split()[1]
            op = op.split(".")[0]
            ie = int(r[ix["Instructions Executed"]] or 0)
            ss = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            by_op[op] += ie
            stall[op] += ss
            tot_i += ie
            tot_s += ss
            hot.append((ss, ie, r[ix["Address"]], src))
        print("=" * 100)
        print(name.strip()[:150])
        print(f"warp instructions executed: {tot_i:,}   stall samples: {tot_s:,}")
        print("opcode           instr%   stall%")
        for op, _ in sorted(stall.items(), key=lambda kv: -kv[1])[:25]:
            print(f"{op:15s} {100*by_op[op]/max(tot_i,1):6.1f}  {100*stall[op]/max(tot_s,1):6.1f}")
        print("hottest instructions (stall samples):")
        for ss, ie, addr, src in sorted(hot, reverse=True)[:25]:
            print(f"{ss:8d} {ie:12d}  {src}")


if __name__ == "__main__":
    main()
