# dominant cfg5 stage (mask 127) under different hand-over knobs
run() { echo "$1: $(env $1 timeout 300 python tools/cfg5_probe.py cfg5 127 x 2>&1 | tail -1 | grep -o "0x1[^ ]*\|.device_ms.: [0-9.]*" | tr '\n' ' ')"; }
for r in 1 2; do
run MOSAIC_DON_PERIOD=1
run MOSAIC_DON_PERIOD=4
run MOSAIC_DON_PERIOD=16
run MOSAIC_DON_DEPTH=2
run MOSAIC_DON_DEPTH=4
run MOSAIC_DEEP_AFTER=1024
run MOSAIC_DEEP_AFTER=16384
run MOSAIC_BACKOFF_NS=512
done
