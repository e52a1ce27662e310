for O in 3,0,1,2,4,5,6 3,0,6,5,4,2,1 0,3,1,2,4,5,6 3,0,2,1,4,5,6 1,2,4,5,6,3,0 3,0,4,5,6,1,2 3,0,1,4,2,5,6 3,1,0,2,4,5,6; do
  echo "order $O: $(MOSAIC_MIN_ORDER=$O timeout 60 python tools/prof_min.py 2>&1 | grep -o "'ksearch_ms': [0-9.]*")"
done
