set -x
free -g | head -2; nproc
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --steps 8 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo bench=$?; cat gpurun_out/bench_n4.json; grep -v -i warn gpurun_out/bench_n4.err | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/multirank_gpu.py 2>&1 | grep '^{' 
