set -x
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_search -s 4 -c 4 -o gpurun_out/prof_min127 python tests/_cfg5_probe.py cfg5 127 nosolve > gpurun_out/ncu_prof_min127.log 2>&1
tail -5 gpurun_out/ncu_prof_min127.log
