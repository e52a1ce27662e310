set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err
tail -c 2500 gpurun_out/bench_r1b.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1b.json 2>&1
tail -c 1500 gpurun_out/bench_ref_r1b.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5_solve.csv python tests/_cfg5_probe.py cfg5 1 > gpurun_out/launches_cfg5_solve.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search -s 6 -c 1 -o gpurun_out/prof_ksearch_min127 python tests/_cfg5_probe.py cfg5 127 nosolve > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out
