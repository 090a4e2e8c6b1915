"""Sum dram bytes / duration of the kernels of the last RK step in an ncu
--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--csv launch list of tools/prof_stage_ns.py; writes the per-stage traffic JSON.
usage: python tools/stage_traffic.py launches.csv nlast out.json"""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14]
hdr = rows[0]
data = collections.OrderedDict()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    key = int(d["ID"])
    e = data.setdefault(key, {"kernel": d["Kernel Name"]})
    unit = d["Metric Unit"]
    v = float(d["Metric Value"].replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1)
    e[d["Metric Name"]] = v * mult
nlast = int(sys.argv[2])
last = list(data.values())[-nlast:]
per_kernel = collections.OrderedDict()
for e in last:
    k = e["kernel"].split("(")[0]
    a = per_kernel.setdefault(k, {"launches": 0, "dram_bytes": 0.0, "us": 0.0})
    a["launches"] += 1
    a["dram_bytes"] += e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
    a["us"] += e.get("gpu__time_duration.sum", 0)
tot = sum(a["dram_bytes"] for a in per_kernel.values())
stages = 3
out = {"source": sys.argv[1], "launches_of_step": nlast, "dram_bytes_per_stage": tot / stages,
       "per_kernel_per_step": per_kernel,
       "note": "ncu --clock-control none, cold-cache per kernel (ncu flushes between kernels); one RK3 step = 3 stages"}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out, indent=1))
