"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit")
    if unit in ("nsecond", "ns"):
        v /= 1e3
    elif unit in ("msecond", "ms"):
        v *= 1e3
    k = d["Kernel Name"]
    c = tot.setdefault(k, [0, 0.0])
    c[0] += 1
    c[1] += v
T = sum(v[1] for v in tot.values())
for k, (n, v) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{k[:70]:70s} n={n:5d} total_us={v:11.1f} avg_us={v / n:9.1f} share={100 * v / T:5.1f}%")
print(f"TOTAL_us={T:.1f}")
