CMD="python bench.py --steps 4 --warmup 3 --no-cpu --no-stall"
timeout 600 $CMD > gpurun_out/plain_launch2.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1e.csv $CMD > gpurun_out/ncu_launch_r1e.log 2>&1; echo ncu1=$?
CMD2="python bench.py --workload gpt125m --steps 3 --warmup 3 --no-cpu --no-stall --no-e2e"
timeout 600 $CMD2 > gpurun_out/plain_la2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"token_hist|select_load|expand_plan|copy_bulk" -s 8 -c 5 -o gpurun_out/prof_loadaware2 $CMD2 > gpurun_out/ncu_la2.log 2>&1; echo ncu2=$?
