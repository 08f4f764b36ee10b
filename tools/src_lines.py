"""Per-CUDA-line totals (instructions, stall samples, excessive shared
wavefronts) from an ncu source page.  usage: src_lines.py rep [sort_col] [n]"""
import csv, subprocess, sys

rep = sys.argv[1]
key = sys.argv[2] if len(sys.argv) > 2 else "Instructions Executed"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
f, h, res = None, None, []
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r[0] == "Line No":
        h = r
    elif h and r[0] not in ("", "Function Name"):
        try:
            res.append((f, r[0], r[1].strip()[:70], float(r[h.index("Instructions Executed")] or 0),
                        float(r[h.index("Warp Stall Sampling (All Samples)")] or 0),
                        float(r[h.index("L1 Wavefronts Shared Excessive")] or 0)))
        except (ValueError, IndexError):
            pass
col = {"Instructions Executed": 3, "stall": 4, "excess": 5}.get(key, 3)
for x in sorted(res, key=lambda x: -x[col])[:n]:
    print(f"{x[0]:12s}{x[1]:>5s} {x[3]:13.0f} {x[4]:8.0f} {x[5]:11.0f}  {x[2]}")
