#!/bin/bash
# GPU-box profiling recipe (B200_PROFILING.md): plain runs first, then ncu.
#   1. launch list of the bench command (our kernels only; per-launch device time)
#   2. one `--set full` capture of the dominant kernel inside the bench command
#   3. one `--set full` capture of the Euler kernel (cfg5 slice)
set -u
OUT=${1:-gpurun_out}
mkdir -p $OUT
BENCH="python bench.py --steps 1 --warmup 1 --time-steps 1000 --no-e2e --no-cpu --no-parity --no-configs"
$BENCH > $OUT/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_blocked|k_minmax" -c 400 --csv \
    --log-file $OUT/launches.csv $BENCH > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?" >> $OUT/ncu_launches.log
BENCH1="python bench.py --steps 1 --warmup 0 --time-steps 64 --no-e2e --no-cpu --no-parity --no-configs"
$BENCH1 > $OUT/bench_tiny.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_blocked -s 1 -c 1 \
    -o $OUT/prof_bench -f $BENCH1 > $OUT/ncu_bench.log 2>&1
echo "bench full capture rc=$?" >> $OUT/ncu_bench.log
python tools/prof_step.py euler > $OUT/prof_plain_euler.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_euler -s 1 -c 1 \
    -o $OUT/prof_euler -f python tools/prof_step.py euler > $OUT/ncu_euler.log 2>&1
echo "euler full capture rc=$?" >> $OUT/ncu_euler.log
# 4. cfg3: the persistent LIN kernel (K2P), 128 steps of the 2^24-cell problem
python tools/prof_step.py lin > $OUT/prof_plain_lin.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_blocked -c 1 \
    -o $OUT/prof_lin -f python tools/prof_step.py lin 16777216 512 > $OUT/ncu_lin.log 2>&1
echo "lin full capture rc=$?" >> $OUT/ncu_lin.log
