set -u
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu"
timeout 900 $B --stall-rounds 3 > gpurun_out/st_diag.json 2> gpurun_out/st_diag.err; echo a=$?
free -g > gpurun_out/free.txt; df -h /dev/shm >> gpurun_out/free.txt
