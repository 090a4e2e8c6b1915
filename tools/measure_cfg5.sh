#!/bin/bash
# The cfg5 measurement package of a round (run on the GPU box from the repo
# root; outputs under gpurun_out/):
#   bench line, ncu launch list of the bench (gpu__time_duration only),
#   per-stage DRAM traffic of one RK step, ncu --set full of the two largest
#   kernels (k_ns_face<1,2> = W=1 flux pass, k_ns_res = RK-stage element kernel).
set -x
O=gpurun_out/m; mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
# the N > 1 code path (DistSolver, NCCL group, per-stage exchange calls) on this one rank
BENCH_FORCE_DIST=1 python bench.py --no-cpu-baseline > $O/bench_forcedist.json 2> $O/bench_forcedist.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_ncu.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/stage_traffic.csv python tools/prof_stage_ns.py > $O/stage.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name regex:k_ns_face --launch-skip 21 --launch-count 1 \
    -o $O/face12 python tools/prof_stage_ns.py > $O/ncu_face.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name regex:k_ns_res --launch-skip 3 --launch-count 1 \
    -o $O/res python tools/prof_stage_ns.py > $O/ncu_res.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name regex:k_tau_grp --launch-skip 0 --launch-count 1 \
    -o $O/tau python tools/prof_tau_ns.py > $O/ncu_tau.log 2>&1
ls -la $O
