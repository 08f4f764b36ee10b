"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): device
time per kernel family and its share.  usage: launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")[:64]
    tot[name] += float(r[ix["Metric Value"]].replace(",", "")) * scale[r[ix["Metric Unit"]]]
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':64s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, v in tot.most_common():
    print(f"{k:64s} {cnt[k]:8d} {v:10.3f} {100 * v / T:6.2f}%")
print(f"{'total':64s} {sum(cnt.values()):8d} {T:10.3f}")
