# specialised vs generic search kernel on the dominant cfg5 stage and the full solve
for r in 1 2; do
  echo "fast    $(timeout 300 python tools/cfg5_probe.py cfg5 127 x 2>&1 | tail -1 | grep -o "0x1[^ ]*\|.device_ms.: [0-9.]*" | tr '\n' ' ')"
  echo "generic $(MOSAIC_GENERIC_KERNEL=1 timeout 300 python tools/cfg5_probe.py cfg5 127 x 2>&1 | tail -1 | grep -o "0x1[^ ]*\|.device_ms.: [0-9.]*" | tr '\n' ' ')"
done
