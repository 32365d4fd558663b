set -x
timeout 900 python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; echo bench=$?; cat gpurun_out/bench_r1b.json; tail -5 gpurun_out/bench_r1b.err
timeout 600 python bench.py --engine vec --no-e2e --no-cpu > gpurun_out/bench_r1b_vec.json 2>&1; cat gpurun_out/bench_r1b_vec.json | tail -2
