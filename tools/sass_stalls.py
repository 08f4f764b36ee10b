"""Stall samples of an ncu report per SASS opcode (which instructions wait, and on what).
usage: sass_stalls.py report.ncu-rep"""
import csv, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
h = None
agg = defaultdict(lambda: defaultdict(float))
cols = ["Warp Stall Sampling (All Samples)", "stall_wait", "stall_math", "stall_short_sb", "stall_long_sb",
        "stall_dispatch", "stall_not_selected", "stall_selected", "stall_mio", "stall_branch_resolving", "Instructions Executed"]
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "Address":
        h = r
        continue
    if h is None or len(r) != len(h):
        continue
    src = r[h.index("Source")].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    for c in cols:
        try:
            agg[op][c] += float(r[h.index(c)] or 0)
        except ValueError:
            pass
tot = sum(v[cols[0]] for v in agg.values())
print(f"{'op':10s} {'all%':>6s} " + " ".join(f"{c.replace('stall_', '')[:8]:>8s}" for c in cols[1:-1]) + "   instr")
for op, v in sorted(agg.items(), key=lambda x: -x[1][cols[0]])[:28]:
    print(f"{op:10s} {100 * v[cols[0]] / tot:6.1f} " + " ".join(f"{100 * v[c] / tot:8.1f}" for c in cols[1:-1]) + f"  {v[cols[-1]]:.3g}")
