timeout 200 python tests/_prof_min.py
timeout 1500 ncu --section SpeedOfLight --section WarpStateStats --section Occupancy --section SchedulerStats --section LaunchStats --section MemoryWorkloadAnalysis --clock-control none --replay-mode application -k regex:k_search -c 1 -o gpurun_out/prof_min127d python tests/_prof_min.py > gpurun_out/ncu_prof_min127d.log 2>&1
tail -3 gpurun_out/ncu_prof_min127d.log
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3
