# Per-config timings, DRAM traffic of every k_search launch of one cfg5 solve, and a
# section capture of the dominant launch (the 7-encoder MIN proof).
set -x
bash tools/bench_all_configs.sh > gpurun_out/all_configs.txt 2>&1; cat gpurun_out/all_configs.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/dram_cfg5_solve.csv \
  python tools/cfg5_probe.py cfg5 1 > /dev/null 2>&1
timeout 1200 ncu --section SpeedOfLight --section WarpStateStats --section Occupancy \
  --section SchedulerStats --section LaunchStats --section MemoryWorkloadAnalysis \
  --section ComputeWorkloadAnalysis --import-source on --clock-control none \
  --replay-mode application -k regex:k_search -c 1 -f -o gpurun_out/prof_min_r1e \
  python tools/prof_min.py > gpurun_out/ncu_prof_min_r1e.log 2>&1; tail -5 gpurun_out/ncu_prof_min_r1e.log
