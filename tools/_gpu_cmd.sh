set -u
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default2.json 2> gpurun_out/bench_default2.err; echo default=$?
bash tools/gpu_recipes.sh sanitize
