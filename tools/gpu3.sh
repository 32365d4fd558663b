set -x
timeout 300 python tools/d2h_probe.py > gpurun_out/d2h_probe.json 2>&1; cat gpurun_out/d2h_probe.json
CMD="python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --engine bulk"
timeout 300 $CMD > gpurun_out/plain_mixtral.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mixtral.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo ncu1=$?
CMD2="python bench.py --workload gpt350m --steps 2 --warmup 3 --no-e2e --no-cpu --engine bulk"
timeout 300 $CMD2 > gpurun_out/plain_gpt350.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_ -s 1 -c 2 -o gpurun_out/prof_pack_bulk $CMD2 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/ncu_full.log
