# ncu target: the cfg5 7-encoder stage_eval; its 5th FIRST launch is the last seeded probe
# (~0.17 s, 25 M nodes): ncu -k regex:k_search_fast_first --launch-skip 4 --launch-count 1
import sys
sys.path.insert(0, '.')
import paper_2605_18710_b200.mosaic as m
pl = m.Planner.from_spec('cfg5')
r = pl.stage_eval(list(range(7)))
print('T', r.stage_time.hex(), r.stats)
