"""Attribute register moves (MOV / IMAD.MOV) and NOPs to CUDA source lines
from an ncu source page.  usage: mov_lines.py rep [n]"""
import csv, subprocess, sys, collections

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
f, h, cur, d = None, None, None, collections.Counter()
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r[0] == "Line No":
        h = r
    elif h and r[0]:
        cur = f"{f}:{r[0]} {r[1].strip()[:60]}"
    elif h and len(r) > 3 and r[2] not in ("...", ""):
        op = r[3].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        if o.startswith(("MOV", "IMAD.MOV", "NOP")):
            try:
                d[(cur, o.split(".")[0])] += float(r[h.index("Instructions Executed")] or 0)
            except ValueError:
                pass
for (line, o), v in d.most_common(n):
    print(f"{v / 1e6:9.1f}M {o:5s} {line}")
