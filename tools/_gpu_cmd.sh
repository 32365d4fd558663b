set -u
mkdir -p gpurun_out
bash tools/gpu_recipes.sh guard
bash tools/gpu_recipes.sh launches
