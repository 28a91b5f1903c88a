"""One-line summary of a bench JSON line: value, e2e, latency, per-kernel us per launch."""
import json, sys
for p in sys.argv[1:]:
    d = json.loads(open(p).read().strip().splitlines()[-1])
    print(p, 'value', round(d['value'], 1), 'e2e', round(d['e2e']['value'], 1), 'lat', round(d.get('latency_ms_per_frame', 0), 4),
          'frac', round(d['roofline']['frac'], 3), {k.split(' ')[0]: round(v['ms_per_launch'] * 1e3, 1) for k, v in d['kernels'].items()})
