set -x
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
for f in "32 24 202" "16 16 302" "16 16 402" "16 24 402" "32 16 202" "32 32 202"; do set -- $f; TUNE_N=268435456 TUNE_V=$1 TUNE_K=$2 TUNE_FAM=$3 timeout 120 python tools/tune.py eo; done > gpurun_out/eo_vk.jsonl 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err
