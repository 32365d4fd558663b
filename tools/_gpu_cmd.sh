set -u
mkdir -p gpurun_out
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_suite.txt 2>&1; echo suite=$?; tail -3 $O/gpu_suite.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo smoke=$?; tail -2 $O/smoke.txt
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_r2b.json 2> $O/bench_r2b.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_r2b_ref.json 2> $O/bench_r2b_ref.err; echo ref=$?
