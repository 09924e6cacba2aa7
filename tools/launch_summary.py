"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: time share per kernel."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    name = r[4].split("(")[0].replace("void ", "").strip()
    v = float(r[14].replace(",", ""))
    unit = r[13]
    ns = v * {"ns": 1, "nsecond": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
    tot[name] += ns
    cnt[name] += 1
all_ns = sum(tot.values())
print(f"{'kernel':70s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:70]:70s} {cnt[k]:8d} {v / 1e6:10.3f} {100 * v / all_ns:6.1f}%")
print(f"{'TOTAL':70s} {sum(cnt.values()):8d} {all_ns / 1e6:10.3f}")
