set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python __graft_entry__.py 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo bench=$?; cat gpurun_out/bench_r1.json; tail -3 gpurun_out/bench_r1.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 300 $CMD > gpurun_out/plain_full.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 2 -c 1 -o gpurun_out/prof_pack_mixtral $CMD > gpurun_out/ncu_full_mixtral.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_full_mixtral.log
