"""Instruction share per code region ("// ---- title" comments) of one kernel.
    python tools/ncu_regions.py report.ncu-rep kernel-regex source.cu"""
import collections, csv, io, re, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv",
                      "--print-source=cuda,sass", "-k", "regex:" + sys.argv[2], "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ix = {}
for j, h in enumerate(hdr):
    ix.setdefault(h, j)
target = sys.argv[3].split("/")[-1]
src = open(sys.argv[3]).read().split("\n")
marks = [(0, "(file head)")]
for n, l in enumerate(src, 1):
    m = re.match(r"\s*// ---- (.*?)-*$", l) or re.match(r"^(?:template.*\n)?.*__(?:device|global)__.*?(\w+)\(", l)
    if m:
        marks.append((n, m.group(1).strip()[:50]))
tot = collections.Counter()
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) < len(hdr) or not r[0] or r[0] == "Line No":
        continue
    try:
        ie = int(r[ix["Instructions Executed"]] or 0)
        ln = int(r[0])
    except ValueError:
        continue
    lab = "(other files)"
    if fname == target:
        lab = [m for n, m in marks if n <= ln][-1]
    tot[lab] += ie
T = sum(tot.values()) or 1
for k, v in tot.most_common():
    print(f"{100 * v / T:5.1f}%  {v:>12,}  {k}")
