import json, sys
for f in sys.argv[1:]:
    for l in open(f):
        try:
            d = json.loads(l)
        except Exception:
            print(l.strip()); continue
        print(d['config'], d['ordering'], d['var'], d['sched']['kind'], d['sched']['tile'], d['sched']['lag'], d['sched'].get('tiling'), d['sched'].get('n_tiles'), d['sched'].get('max_reach'),
              '%.1f us/sweep %.1f Gvups %.0f GB/s frac %.3f' % (d['us_per_sweep'], d['gvups'], d['gbs'], d['frac']))
