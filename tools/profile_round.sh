#!/bin/bash
# GPU-box profiling recipe (B200_PROFILING.md): plain runs first, then ncu.
#   1. launch list of the bench command (our kernels only; per-launch device time)
#   2. one `--set full` capture of the dominant kernel on a bench-shaped slice
set -u
OUT=${1:-gpurun_out}
mkdir -p $OUT
BENCH="python bench.py --steps 1 --warmup 1 --time-steps 1000 --no-e2e --no-cpu --no-parity"
$BENCH > $OUT/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_blocked|k_minmax" -c 400 --csv \
    --log-file $OUT/launches.csv $BENCH > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?" >> $OUT/ncu_launches.log
python tools/prof_step.py eo > $OUT/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_blocked -s 1 -c 1 \
    -o $OUT/prof_eo python tools/prof_step.py eo > $OUT/ncu_eo.log 2>&1
echo "full capture rc=$?" >> $OUT/ncu_eo.log
