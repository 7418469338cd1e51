"""Readable summary of a bench.py JSON line."""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print('value', round(d['value'], 1), d['unit'], 'ms/step', round(d['ms_per_step'], 1), 'pipelined', d.get('pipelined'))
print('full_inverse', d['full_inverse'])
r = d['roofline']; print('roofline', r['kernel'], round(r['frac'], 3), r['bound'], round(r['achieved'], 2), r['unit'], 'traffic', r.get('traffic'))
print('e2e', {k: d['e2e'][k] for k in ('value', 'h2d_bytes_per_step', 'd2h_bytes_per_step', 'ms_per_step')} if d.get('e2e') else None)
print('cpu', d['cpu_baseline']['value'] if d.get('cpu_baseline') else None, 'launches', d['gpu_launches'], 'clocks', d['clocks'])
print('stages', {k: round(v, 1) for k, v in d['stages_ms_per_step'].items()})
print('methods', d['method_counts'], d['iters_hist'])
for k, v in list(d['kernels'].items())[:12]:
    print('  ', k, round(v['ms_total_per_step'], 2), v['launches_per_step'], round(v.get('frac', 0), 3))
for k, v in d.get('configs', {}).items():
    for x in v:
        if isinstance(v[x], dict) and 'updates_per_s' in v[x]:
            rr = v[x].get('roofline') or {}
            print(k, x, round(v[x]['updates_per_s']), 'pipe' if v[x].get('pipelined') else 'seq', rr.get('kernel'), round(rr.get('frac', 0), 3),
                  'cpu', round(v['cpu_baseline']['value']) if 'cpu_baseline' in v else None)
if d.get('leo_campaign'):
    print('leo', round(d['leo_campaign']['value']), d['leo_campaign']['table'])
