mkdir -p gpurun_out
B=$PWD/paper_2604_06947_b200/build
T="timeout 300 python tools/tune.py eo"
{
FQNM_LIBPATH=$PWD/paper_2604_06947_b200/libfqnm.so TUNE_N=268435456 TUNE_V=32 TUNE_K=32 TUNE_FAM=202 $T | sed "s/^/default /"
FQNM_LIBPATH=$B/libfqnm_fsx.so TUNE_N=268435456 TUNE_V=32 TUNE_K=32 TUNE_FAM=202,302 $T | sed "s/^/fsx /"
FQNM_LIBPATH=$B/libfqnm_fsx.so TUNE_N=268435456 TUNE_V=64 TUNE_K=32,48,64 TUNE_FAM=102,202 $T | sed "s/^/fsx /"
FQNM_LIBPATH=$B/libfqnm_fsx.so TUNE_N=268435456 TUNE_V=16 TUNE_K=16,24 TUNE_FAM=302,402 $T | sed "s/^/fsx /"
FQNM_LIBPATH=$B/libfqnm_evx.so TUNE_N=268435456 TUNE_V=64 TUNE_K=32,48 TUNE_FAM=102,202 $T | sed "s/^/evx /"
FQNM_LIBPATH=$B/libfqnm_evx.so TUNE_N=268435456 TUNE_V=32 TUNE_K=32 TUNE_FAM=302 $T | sed "s/^/evx /"
} > gpurun_out/sweep_occ.log 2>&1
