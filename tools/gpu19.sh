CMD="python bench.py --workload gpt350m --engine crc --steps 2 --warmup 3 --no-cpu --no-stall --no-e2e"
timeout 300 $CMD > gpurun_out/plain_crc.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pack_crc|crc_fold|crc_final" -s 3 -c 3 -o gpurun_out/prof_crc $CMD > gpurun_out/ncu_crc.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_crc.log
