# A/B of library variants in _var/lib*.so on the dominant cfg5 stage (mask 127), 2 rounds
for r in 1 2; do
for L in _var/lib*.so; do
  echo "== $L"; MOSAIC_LIB=$L timeout 300 python tools/cfg5_probe.py cfg5 127 x 2>&1 | tail -1 | cut -c1-60,200-
done; done
