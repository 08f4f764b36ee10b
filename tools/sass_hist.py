"""Per-opcode histogram of an ncu source page (SASS): instructions executed,
stall samples and excessive shared wavefronts.  usage: sass_hist.py a.ncu-rep [b.ncu-rep]"""
import csv, subprocess, sys, collections


def hist(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h = rows[0]
    ix = {k: h.index(k) for k in ("Source", "Instructions Executed", "Warp Stall Sampling (All Samples)",
                                  "L1 Wavefronts Shared Excessive")}
    d = collections.defaultdict(lambda: [0, 0, 0])
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        op = r[ix["Source"]].split()
        if not op:
            continue
        o = op[0] if not op[0].startswith("@") else op[1]
        o = o.split(".")[0] if o.startswith(("DFMA", "DADD", "DMUL", "IMAD", "IADD3", "LOP3", "SHF")) else o
        for j, k in enumerate(("Instructions Executed", "Warp Stall Sampling (All Samples)",
                               "L1 Wavefronts Shared Excessive")):
            try:
                d[o][j] += float(r[ix[k]])
            except ValueError:
                pass
    return d


reps = [hist(r) for r in sys.argv[1:]]
keys = sorted(set().union(*reps), key=lambda k: -max(r.get(k, [0])[0] for r in reps))
print(f"{'opcode':28s}" + "".join(f"{'inst':>14s}{'stall':>9s}{'exc_wf':>12s}" for _ in reps))
for k in keys[:45]:
    print(f"{k:28s}" + "".join(f"{r.get(k, [0,0,0])[0]:14.0f}{r.get(k, [0,0,0])[1]:9.0f}{r.get(k, [0,0,0])[2]:12.0f}" for r in reps))
