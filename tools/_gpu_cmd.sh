set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29561 tools/multirank_gpu.py --config3 --ranks-per-proc 2 > $O/mr_c3_nccl4x2.txt 2>&1; echo mr_nccl=$?
grep '^{' $O/mr_c3_nccl4x2.txt
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29564 bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench_n4.json 2> $O/bench_n4.err; echo bench4=$?
free -g > $O/free_after.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29565 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > $O/bench_n4_ref.json 2> $O/bench_n4_ref.err; echo ref4=$?
