"""Print selected 'details' metrics of every kernel in an ncu report.
    python tools/ncu_details.py report.ncu-rep [regex]"""
import csv, io, re, subprocess, sys
KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Block Limit Registers", "Block Limit Shared Mem",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Issue Slots Busy", "Executed Instructions",
        "Grid Size", "Dynamic Shared Memory Per Block", "Mem Busy", "Max Bandwidth",
        "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
cur = None
for r in rows[1:]:
    name = r[ix["Kernel Name"]]
    if pat and not pat.search(name):
        continue
    key = (r[ix["ID"]], name)
    if key != cur:
        cur = key
        print(f"--- [{r[ix['ID']]}] {name[:110]}")
    if r[ix["Metric Name"]] in KEEP:
        print(f"    {r[ix['Metric Name']]:40s} {r[ix['Metric Value']]:>14s} {r[ix['Metric Unit']]}")
