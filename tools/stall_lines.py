"""CUDA lines ranked by one stall reason (ncu source page).  usage: stall_lines.py rep reason [n]"""
import csv, subprocess, sys

rep, reason = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
f, h, res, tot = None, None, [], 0.0
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r[0] == "Line No":
        h = r
    elif h and r[0] not in ("", "Function Name"):
        try:
            v = float(r[h.index(reason)] or 0)
        except (ValueError, IndexError):
            continue
        tot += v
        res.append((v, f, r[0], r[1].strip()[:80]))
for v, f, ln, src in sorted(res, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  {f}:{ln}  {src}")
