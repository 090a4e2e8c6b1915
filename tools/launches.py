"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
t = collections.defaultdict(float)
c = collections.Counter()
for r in rows[start + 1:]:
    if len(r) > iv:
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        name = r[ik].split("(")[0]
        t[name] += v
        c[name] += 1
tot = sum(t.values())
for k, v in sorted(t.items(), key=lambda x: -x[1]):
    print(f"{k:50s} n={c[k]:5d} total_us={v / 1000:10.1f} avg_us={v / 1000 / c[k]:8.1f} share={v / tot * 100:5.1f}%")
