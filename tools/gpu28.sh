set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python __graft_entry__.py
timeout 900 python bench.py > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err; echo bench=$?; cat gpurun_out/bench_r1d.json
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-stall"
timeout 300 $CMD > gpurun_out/plain_full2.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:copy_bulk -s 2 -c 1 -o gpurun_out/prof_pack_mixtral_v2 $CMD > gpurun_out/ncu_full_mixtral2.log 2>&1; echo ncu=$?
