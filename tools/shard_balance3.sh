for r in 0 2 5; do MOSAIC_TRACE=1 MOSAIC_SHARD_SIM=$r/8 timeout 60 python tools/prof_min.py 2>&1 | grep "MIN" | cut -c1-160; done
MOSAIC_TRACE=1 timeout 60 python tools/prof_min.py 2>&1 | grep "MIN" | cut -c1-160
