# dominant cfg5 stage (mask 127) under hand-over knob variants (current kernels)
run() { echo "$1: $(env $1 timeout 300 python tools/cfg5_probe.py cfg5 127 x 2>&1 | tail -1 | grep -o "0x1[^ ]*\|.device_ms.: [0-9.]*" | tr '\n' ' ')"; }
for r in 1 2; do
run MOSAIC_DON_PERIOD=4
run MOSAIC_DON_PERIOD=8
run MOSAIC_DEEP_AFTER=65536
run MOSAIC_BACKOFF_NS=1024
run MOSAIC_BACKOFF_NS=4096
done
