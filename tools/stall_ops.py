"""Stall reasons by opcode of the stalled instruction (ncu source page, SASS).
usage: stall_ops.py rep [n]"""
import csv, subprocess, sys, collections

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
reasons = ["stall_selected", "stall_wait", "stall_short_sb", "stall_math", "stall_not_selected", "stall_mio",
           "stall_dispatch", "stall_barrier", "stall_long_sb", "stall_branch_resolving", "stall_no_inst"]
ix = {r: h.index(r) for r in reasons}
d = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in rows[1:]:
    if len(r) != len(h):
        continue
    op = r[1].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    for k, i in ix.items():
        try:
            v = float(r[i] or 0)
        except ValueError:
            continue
        d[o][k] += v
        tot[k] += v
T = sum(tot.values())
print(f"{'opcode':10s}" + "".join(f"{k[6:14]:>9s}" for k in reasons) + "   total%")
for o in sorted(d, key=lambda o: -sum(d[o].values()))[:int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    print(f"{o:10s}" + "".join(f"{100 * d[o][k] / T:9.1f}" for k in reasons) + f"   {100 * sum(d[o].values()) / T:6.1f}")
print(f"{'ALL':10s}" + "".join(f"{100 * tot[k] / T:9.1f}" for k in reasons))
