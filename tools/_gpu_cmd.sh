mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_e2e.py -q -x > gpurun_out/t.log 2>&1; echo EXIT $? >> gpurun_out/t.log
for r in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_ramp$r.log 2>&1; done
