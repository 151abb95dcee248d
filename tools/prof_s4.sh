#!/bin/bash
# session-4 captures: cfg3 (K2P LIN and K2 LIN) and the Euler kernel, --set full with source
set -u
OUT=${1:-gpurun_out}
mkdir -p $OUT
python tools/prof_step.py lin > $OUT/s4_plain_lin.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_blocked -c 1 \
    -o $OUT/s4_prof_lin -f python tools/prof_step.py lin > $OUT/s4_ncu_lin.log 2>&1
echo "lin rc=$?" >> $OUT/s4_ncu_lin.log
python tools/prof_step.py euler > $OUT/s4_plain_euler.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_euler -s 1 -c 1 \
    -o $OUT/s4_prof_euler -f python tools/prof_step.py euler > $OUT/s4_ncu_euler.log 2>&1
echo "euler rc=$?" >> $OUT/s4_ncu_euler.log
