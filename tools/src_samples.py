"""Warp-stall samples of an ncu report aggregated per CUDA source line and per file.
usage: src_samples.py report.ncu-rep [n]"""
import csv, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
f, h, lines, files = None, None, [], defaultdict(float)
tot = 0.0
for r in csv.reader(out):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        f = r[1].split("/")[-1]
    elif r[0] == "Line No":
        h = r
    elif h and r[0] not in ("", "Function Name"):
        try:
            v = float(r[h.index("Warp Stall Sampling (All Samples)")] or 0)
            ins = float(r[h.index("Instructions Executed")] or 0)
        except (ValueError, IndexError):
            continue
        tot += v
        files[f] += v
        lines.append((v, ins, f, r[0], r[1].strip()[:90]))
for k, v in sorted(files.items(), key=lambda x: -x[1]):
    print(f"{100 * v / tot:5.1f}%  {k}")
print()
for v, ins, f, ln, src in sorted(lines, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  {ins:12.0f}  {f}:{ln}  {src}")
