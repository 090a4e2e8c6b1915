"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
LAST = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # only the last LAST launches (one bench step)
hdr = None
tot = collections.OrderedDict()
launches = []
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
    launches.append((d["Kernel Name"], v))
for k, v in launches[-LAST:] if LAST else launches:
    c = tot.setdefault(k, [0, 0.0])
    c[0] += 1
    c[1] += v
T = sum(v[1] for v in tot.values())
for k, (n, v) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{k[:70]:70s} n={n:5d} total_us={v:11.1f} avg_us={v / n:9.1f} share={100 * v / T:5.1f}%")
print(f"TOTAL_us={T:.1f}")
