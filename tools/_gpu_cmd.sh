set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 1800 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider > $O/multigpu_n2.txt 2>&1; echo mg=$?; tail -2 $O/multigpu_n2.txt
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29571 bench.py --gpus 2 --steps 20 --warmup 5 > $O/bench_n2.json 2> $O/bench_n2.err; echo bench2=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29572 bench.py --impl reference --gpus 2 --steps 20 --warmup 5 > $O/bench_n2_ref.json 2> $O/bench_n2_ref.err; echo ref2=$?
