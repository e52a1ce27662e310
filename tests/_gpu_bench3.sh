set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err
tail -c 2600 gpurun_out/bench_r1c.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5_solve_c.csv python tests/_cfg5_probe.py cfg5 1 > gpurun_out/launches_cfg5_solve_c.log 2>&1
timeout 900 ncu --section SpeedOfLight --section WarpStateStats --section Occupancy --section SchedulerStats --section LaunchStats --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section SourceCounters --import-source on --clock-control none -k regex:k_search -s 3 -c 3 -o gpurun_out/prof_min127c python tests/_cfg5_probe.py cfg5 127 nosolve > gpurun_out/ncu_prof_min127c.log 2>&1
tail -2 gpurun_out/ncu_prof_min127c.log
