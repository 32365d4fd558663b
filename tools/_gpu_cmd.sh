set -u
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu"
timeout 900 $B > gpurun_out/st_default.json 2> gpurun_out/st_default.err; echo a=$?
timeout 900 $B --stall-no-persist > gpurun_out/st_nopersist.json 2> gpurun_out/st_nopersist.err; echo b=$?
timeout 900 $B --persist-threads 4 > gpurun_out/st_t4.json 2> gpurun_out/st_t4.err; echo c=$?
timeout 900 $B --engine bulk > gpurun_out/st_bulk.json 2> gpurun_out/st_bulk.err; echo d=$?
