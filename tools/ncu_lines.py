"""Per-CUDA-source-line instruction / stall shares of one kernel in an ncu report.
    python tools/ncu_lines.py report.ncu-rep kernel-regex [top]"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv",
                      "--print-source=cuda,sass", "-k", "regex:" + sys.argv[2], "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ix = {}
for j, h in enumerate(hdr):
    ix.setdefault(h, j)
res = []
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) < len(hdr) or not r[0] or r[0] == "Line No":
        continue
    try:
        ie = int(r[ix["Instructions Executed"]] or 0)
        ss = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    res.append((ie, ss, f"{fname}:{r[0]}", r[1][:95]))
tot = sum(x[0] for x in res) or 1
tots = sum(x[1] for x in res) or 1
print(f"warp instructions {tot:,}  stall samples {tots:,}")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
for ie, ss, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100*ie/tot:5.1f}% instr {100*ss/tots:5.1f}% stall  {ln:18s} {src}")
