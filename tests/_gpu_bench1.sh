set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err
tail -c 3000 gpurun_out/bench_r1a.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tests/_cfg5_probe.py cfg4 7,15,56 nosolve > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_search -s 2 -c 2 -o gpurun_out/prof_ksearch python tests/_cfg5_probe.py cfg5 31 nosolve > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
