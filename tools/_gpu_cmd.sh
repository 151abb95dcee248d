mkdir -p gpurun_out
python tools/micro.py r02 > gpurun_out/micro.log 2>&1; cp profiles/r02_micro.json gpurun_out/ 2>/dev/null
B=$PWD/paper_2604_06947_b200/build
{
for v in default linstream; do
  if [ $v = default ]; then L=$PWD/paper_2604_06947_b200/libfqnm.so; else L=$B/libfqnm_$v.so; fi
  FQNM_LIBPATH=$L TUNE_V=32 TUNE_K=64,96,128 TUNE_FAM=202 timeout 300 python tools/tune.py lin | sed "s/^/$v /"
done
} > gpurun_out/sweep_lin.log 2>&1
timeout 600 python tools/bench_configs.py cfg1 cfg2 cfg3 ens1 cfg5 > gpurun_out/configs.log 2>&1
