#!/bin/bash
# The GPU command lines behind profiles/ (one recipe per gpurun call, outputs in gpurun_out/):
#
#   gpurun --timeout 1500 -- 'bash tools/gpu_recipes.sh validate'
#   gpurun --gpus 4 --timeout 1500 -- 'bash tools/gpu_recipes.sh scale 4'
#
# Every ncu capture runs only after the same command exited 0 without ncu, on one GPU.
set -u
mkdir -p gpurun_out
O=gpurun_out
recipe=${1:-validate}

case "$recipe" in
  validate)   # GPU parity suite, smoke, default bench line
    timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
    timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?; cat $O/bench.json
    ;;
  launches)   # per-launch list of the bench's kernels (share of the step)
    CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-stall --e2e-steps 5"
    timeout 600 $CMD > $O/plain_launch.log 2>&1 && \
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo ncu=$?
    ;;
  profile_pack)   # full ncu capture of one Mixtral-rank pack launch (roofline traffic)
    CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-stall"
    timeout 300 $CMD > $O/plain_pack.log 2>&1 && \
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:copy_bulk \
        -s 2 -c 1 -o $O/prof_pack $CMD > $O/ncu_pack.log 2>&1; echo ncu=$?
    ;;
  profile_unpack)   # full ncu capture of one Mixtral-rank unpack (restore scatter) launch
    CMD="python tools/pack_variants.py --unpack-only"
    timeout 600 $CMD > $O/unpack.json 2>&1 && \
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:copy_bulk \
        -s 6 -c 1 -o $O/prof_unpack $CMD > $O/ncu_unpack.log 2>&1; echo ncu=$?
    ;;
  variants)   # pack engine variants vs the library baseline, unpack
    timeout 900 python tools/pack_variants.py > $O/pack_variants.json 2>&1; cat $O/pack_variants.json
    ;;
  profile_loadaware)   # load-aware checkpoint kernels (GPT-MoE 125M-8E)
    CMD="python bench.py --workload gpt125m --steps 3 --warmup 3 --no-cpu --no-stall --no-e2e"
    timeout 600 $CMD > $O/plain_la.log 2>&1 && \
      timeout 900 ncu --set full --clock-control none --import-source on \
        -k regex:"token_hist|select_load|expand_plan|copy_bulk|pack_crc|crc_fold|crc_final" -s 8 -c 8 \
        -o $O/prof_loadaware $CMD > $O/ncu_la.log 2>&1; echo ncu=$?
    ;;
  profile_crc)   # the CRC-computing pack (GPT-MoE 350M-16E)
    CMD="python bench.py --workload gpt350m --engine crc --steps 2 --warmup 3 --no-cpu --no-stall --no-e2e"
    timeout 300 $CMD > $O/plain_crc.log 2>&1 && \
      timeout 900 ncu --set full --clock-control none --import-source on \
        -k regex:"pack_crc|crc_fold|crc_final" -s 3 -c 3 -o $O/prof_crc $CMD > $O/ncu_crc.log 2>&1
    echo ncu=$?
    ;;
  crc_ab)   # CRC-computing pack vs plain pack (Mixtral rank 0), CRC parity tests, ncu of pack_crc
    timeout 900 python -m pytest tests -m gpu -x -q -k "crc or restore" 2>&1 | tail -3
    for e in crc bulk crc; do
      timeout 600 python bench.py --engine $e --steps 10 --warmup 3 --no-e2e --no-cpu --no-stall \
        > $O/bench_$e.json 2> $O/bench_$e.err; echo $e=$?; cat $O/bench_$e.json
    done
    CMD="python bench.py --engine crc --steps 2 --warmup 3 --no-e2e --no-cpu --no-stall"
    timeout 1200 ncu --set full --clock-control none --import-source on \
      -k regex:"pack_crc|crc_fold|crc_final" -s 3 -c 3 -o $O/prof_crc $CMD > $O/ncu_crc.log 2>&1
    echo ncu=$?
    ;;
  guard)   # bounds evidence without compute-sanitizer (closed on this pool): guard bands
           # around every output + the debug library's device-side invariant checks
    PEC_LIB=debug timeout 600 python tools/guard_kernels.py > $O/guard_debug.txt 2>&1; echo guard_debug=$?
    timeout 600 python tools/guard_kernels.py > $O/guard_release.txt 2>&1; echo guard_release=$?
    PEC_LIB=debug timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider \
      > $O/gpu_suite_debug_lib.txt 2>&1; echo suite_debug=$?
    tail -n 2 $O/guard_debug.txt $O/guard_release.txt $O/gpu_suite_debug_lib.txt
    ;;
  host_link)   # pinned D2H / push probes
    timeout 300 python tools/d2h_probe.py > $O/d2h_probe.json 2>&1; cat $O/d2h_probe.json
    timeout 300 python tools/d2h_push_probe.py > $O/d2h_push_probe.json 2>&1
    ;;
  stall_law)   # the reference's stall law vs measured stalls over an F&B sweep (Mixtral rank)
    timeout 900 python tools/stall_law_probe.py > $O/stall_law.json 2> $O/stall_law.err; cat $O/stall_law.json
    ;;
  chain)   # config 5: PEC chain + node fault + restore + K sweep
    timeout 1200 python tools/restore_chain.py --k 1 > $O/restore_chain_k1.json 2> $O/restore_chain.err
    echo chain=$?
    ;;
  scale)   # N-GPU bench (weak scaling), multi-process checks, reference arm
    N=${2:-2}
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus $N \
      > $O/bench_n$N.json 2> $O/bench_n$N.err; echo bench=$?; cat $O/bench_n$N.json
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29552 tools/multirank_gpu.py 2>&1 | grep '^{'
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29553 bench.py --impl reference --gpus $N \
      --steps 2 --warmup 1 2>/dev/null | tail -1 > $O/bench_n${N}_ref.json
    ;;
  restore)   # restore throughput (26.1 GB from /dev/shm storage, device / host verify)
    timeout 900 python tools/restore_bench.py > $O/restore_bench_dev.json
    timeout 900 python tools/restore_bench.py --verify host > $O/restore_bench_host.json
    timeout 600 python tools/register_probe.py --gb 8 > $O/register_probe.json
    ;;
  host)   # host-memory / tmpfs ceilings of the persist tier (run with gpurun --gpus 4)
    (lscpu; nvidia-smi topo -m) > $O/host_topo.txt 2>&1
    timeout 600 python tools/host_probe.py --gb 4 --ranks 4 --threads 8 > $O/host_probe.json
    ;;
  recycle_ab)   # N=4 bench with and without persist-file recycling (gpurun --gpus 4)
    timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 4 --steps 20 --warmup 5 \
      > $O/bench_n4_recycle.json
    timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 4 --steps 5 --warmup 3 \
      --no-cpu --no-recycle > $O/bench_n4_norecycle.json
    ;;
  soak)   # the GPU suite N times (flake hunting); prints one summary line per run
    N=${2:-10}
    for i in $(seq 1 $N); do
      timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed|^E " | head -6
    done
    ;;
  *)
    echo "unknown recipe: $recipe" >&2; exit 2 ;;
esac
