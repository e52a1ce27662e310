# round-end evidence: gpu tests, smoke, bench (ours + reference arm), launch list, DRAM list,
# per-config timings
bash tools/gpu_round_check.sh
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/dram_cfg5_solve.csv \
  python tools/cfg5_probe.py cfg5 1 > /dev/null 2>&1
bash tools/bench_all_configs.sh > gpurun_out/all_configs.txt 2>&1; cat gpurun_out/all_configs.txt
