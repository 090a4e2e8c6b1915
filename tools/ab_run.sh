#!/bin/bash
# A/B timing of kernel variants on the GPU box: tools/ab_run.sh name1 name2 ...
# (each paper_2210_03523_b200/variants/libdgtau_<name>.so), then compares states.
mkdir -p gpurun_out/ab
for v in "$@"; do
  DGTAU_SO=paper_2210_03523_b200/variants/libdgtau_$v.so timeout 600 python tools/kernel_times.py --steps 2 --save /tmp/ab_$v.pt ${AB_ARGS} > gpurun_out/ab/$v.log 2>&1
  echo "== $v"; head -n 12 gpurun_out/ab/$v.log
done
python - "$@" <<'PY'
import sys, torch
ref = torch.load(f"/tmp/ab_{sys.argv[1]}.pt")
for v in sys.argv[2:]:
    x = torch.load(f"/tmp/ab_{v}.pt")
    print(v, "max|d|/max|ref| vs", sys.argv[1], ((x - ref).abs().max() / ref.abs().max()).item(), "bitwise", torch.equal(x, ref))
PY
