set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_suite3.txt 2>&1; echo suite=$?; tail -2 $O/gpu_suite3.txt
timeout 1500 python tools/restore_chain.py --k 1 --verify device > $O/restore_chain_device3.json 2> $O/restore_chain_device3.err; echo chain=$?
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_r2c.json 2> $O/bench_r2c.err; echo bench=$?
