set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
MOSAIC_TRACE=1 timeout 300 python tests/_cfg5_probe.py cfg5 63,127 nosolve 2>&1 | grep -v "kernel=[0-9]\.\|kernel=[0-9][0-9]\.[0-9]*ms" | tail -12
timeout 900 ncu --section SpeedOfLight --section WarpStateStats --section Occupancy --section SchedulerStats --section LaunchStats --section MemoryWorkloadAnalysis --clock-control none -k regex:k_search -s 4 -c 4 -o gpurun_out/prof_min127b python tests/_cfg5_probe.py cfg5 127 nosolve > gpurun_out/ncu_prof_min127b.log 2>&1
tail -3 gpurun_out/ncu_prof_min127b.log
