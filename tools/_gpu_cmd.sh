mkdir -p gpurun_out
B=$PWD/paper_2604_06947_b200/build
for v in default cap2 cap2dual cap4dual dual; do
  if [ $v = default ]; then L=$PWD/paper_2604_06947_b200/libfqnm.so; else L=$B/libfqnm_$v.so; fi
  FQNM_LIBPATH=$L timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_$v.log 2>&1
done
