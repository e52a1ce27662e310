# per-search counters of the small configs: nodes / leaves / kernel time per device search
import sys
sys.path.insert(0, '.')
import paper_2605_18710_b200.mosaic as m
for spec in sys.argv[1:] or ['cfg1', 'cfg2']:
    pl = m.Planner.from_spec(spec)
    pl.solve()
    pl.reset_counters()
    r = pl.solve()
    c = pl.counters()
    n = max(1, c['ksearch_launches'])
    print(spec, 'searches', n, 'k_search us/search %.1f' % (c['ksearch_ms'] * 1e3 / n),
          'device span us/search %.1f' % (c['device_ms'] * 1e3 / n),
          'nodes', r.trace.nodes if hasattr(r.trace, 'nodes') else None,
          'leaves', r.trace.leaves)
