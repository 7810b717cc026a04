"""Summarise an ncu launch list (gpu__time_duration.sum CSV): per-kernel mean
time and share of the total.  usage: python tools/launch_summary.py FILE.csv [skip_first_n]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[h + 1:]:
    if len(r) > vi:
        try:
            agg[r[ki][:70]].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
n_iter = max(len(v) for v in agg.values())
tot = sum(sum(v) for k, v in agg.items() if len(v) >= n_iter // 2)
print(f"{'kernel':70s} {'n':>5s} {'mean us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    s = sum(v) / tot if len(v) >= n_iter // 2 else float("nan")
    print(f"{k:70s} {len(v):5d} {sum(v) / len(v) / 1000:9.1f} {s:6.1%}")
print(f"per-iteration sum of recurring kernels: {tot / n_iter / 1000:.1f} us")
