# one deterministic MIN search: the 7-encoder cfg5 stage proved at T* (for ncu)
import sys
sys.path.insert(0, '.')
import paper_2605_18710_b200.mosaic as m
pl = m.Planner.from_spec('cfg5')
mods = [0, 1, 2, 3, 4, 5, 6]
t = pl.stage_min(mods, float.fromhex('0x1.77e16c9919003p-4'), restart=False)
print('T*', t.hex(), pl.counters())
