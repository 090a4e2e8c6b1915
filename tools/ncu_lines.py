"""Per-source-line aggregation of an ncu --page source --print-source cuda,sass
CSV: warp-stall samples and executed warp instructions per CUDA line."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur_file, cur_line, cur_src = None, None, None
hdr = None
samp = collections.Counter()
inst = collections.Counter()
src = {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iss = hdr.index("Warp Stall Sampling (All Samples)")
        iex = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= iex:
        continue
    if r[0]:
        cur_line, cur_src = int(r[0]), r[1]
        src[(cur_file, cur_line)] = cur_src
        continue
    try:
        samp[(cur_file, cur_line)] += int(r[iss])
        inst[(cur_file, cur_line)] += int(r[iex])
    except ValueError:
        pass
ts, ti = sum(samp.values()), sum(inst.values())
print(f"total samples {ts}, warp instr {ti}")
for k, v in samp.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{v / ts * 100:5.1f}% samp {inst[k] / ti * 100:5.1f}% inst  {k[0]}:{k[1]}  {src[k].strip()[:90]}")
