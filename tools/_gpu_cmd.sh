mkdir -p gpurun_out
for r in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_dual$r.log 2>&1
FQNM_LIBPATH=$PWD/paper_2604_06947_b200/build/libfqnm_nodual.so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > gpurun_out/bench_nodual$r.log 2>&1
done
