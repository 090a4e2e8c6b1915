"""Summarise an ncu --set full report into a small JSON (per kernel: duration,
DRAM bytes, occupancy, IPC, stall breakdown, instruction mix) for profiles/.

usage: python tools/ncu_summary.py report.ncu-rep out.json
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, out):
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = raw[0], raw[1]
    res = []
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))

        def num(k):
            try:
                return float(d[k].replace(",", ""))
            except (KeyError, ValueError):
                return None

        def scaled_bytes(k):
            v = num(k)
            unit = u.get(k, "byte")
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return None if v is None else v * mult

        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(k) for k in hdr
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        stalls = {k: v for k, v in sorted(stalls.items(), key=lambda x: -(x[1] or 0)) if v}
        dur = num("gpu__time_duration.sum")
        res.append({
            "kernel": d.get("Kernel Name"),
            "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
            "duration_us": (dur * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(
                u.get("gpu__time_duration.sum"), 1.0)) if dur else dur,
            "dram_read_bytes": scaled_bytes("dram__bytes_read.sum"),
            "dram_write_bytes": scaled_bytes("dram__bytes_write.sum"),
            "registers": num("launch__registers_per_thread"),
            "achieved_occupancy_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "ipc": num("sm__inst_executed.avg.per_cycle_active"),
            "warp_instructions": num("smsp__inst_executed.sum"),
            "fp64_pipe_pct": num("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
            "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "stall_samples": dict(list(stalls.items())[:8]),
        })
    # instruction mix from the SASS source page (first kernel)
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    try:
        h = src[1]
        isrc, iex = h.index("Source"), h.index("Instructions Executed")
        mix = collections.Counter()
        for r in src[2:]:
            try:
                n = int(r[iex])
            except (ValueError, IndexError):
                continue
            op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip())
            op = op.split()[0].split(".")[0] if op else ""
            mix[op] += n
        tot = sum(mix.values())
        res[0]["sass_mix_pct"] = {k: round(100 * v / tot, 1) for k, v in mix.most_common(14)}
    except Exception:
        pass
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
