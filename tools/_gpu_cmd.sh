set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 1500 python tools/restore_chain.py --k 1 --verify device > $O/restore_chain_device2.json 2> $O/restore_chain_device2.err; echo chain=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_suite2.txt 2>&1; echo suite=$?; tail -2 $O/gpu_suite2.txt
