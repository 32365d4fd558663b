set -u
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi -L > $O/gpus4.txt; free -g >> $O/gpus4.txt; nproc >> $O/gpus4.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29561 tools/multirank_gpu.py --config3 --ranks-per-proc 2 > $O/mr_c3_nccl4x2.txt 2>&1; echo mr_nccl=$?
grep '^{' $O/mr_c3_nccl4x2.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29562 tools/multirank_gpu.py --config3 --backend gloo > $O/mr_c3_gloo8.txt 2>&1; echo mr_gloo8=$?
grep '^{' $O/mr_c3_gloo8.txt
PEC_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 \
  --master-addr 127.0.0.1 --master-port 29563 bench.py --gpus 8 --workload gpt350m --steps 3 \
  --warmup 3 --stall-checkpoints 4 --i-ckpt 2 --stall-rounds 1 --fb-ms 20 --no-cpu \
  > $O/bench_n8_path.json 2> $O/bench_n8_path.err; echo bench8=$?
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29564 bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench_n4.json 2> $O/bench_n4.err; echo bench4=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29565 bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > $O/bench_n4_ref.json 2> $O/bench_n4_ref.err; echo ref4=$?
