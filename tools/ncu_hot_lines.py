"""Top source lines of an ncu report by stall samples and executed
instructions (ncu --page source --print-source cuda,sass).
usage: python tools/ncu_hot_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur_file = None
agg = {}
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue  # keep source-line rows only (sass rows have an address)
    try:
        samp = int(r[4] or 0)
        inst = int(r[7] or 0)
    except ValueError:
        continue
    k = (cur_file, r[0], r[1][:90])
    a = agg.setdefault(k, [0, 0])
    a[0] += samp
    a[1] += inst
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:N]:
    print(f"{100 * v[0] / tot_s:5.1f}% smp {100 * v[1] / tot_i:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
