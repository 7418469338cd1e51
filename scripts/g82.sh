mkdir -p gpurun_out
timeout 2400 python bench.py --no-cpu --no-e2e --steps 2 --warmup 1 > gpurun_out/g82_bench.json 2> gpurun_out/g82_bench.err; echo "bench rc=$?"; tail -5 gpurun_out/g82_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/g82_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['pipelined'], d['pipeline_candidates_ms'], d['roofline']['frac'])
for k,c in d['configs'].items():
    for m,v in c.items():
        if isinstance(v,dict) and 'updates_per_s' in v:
            print(k,m,round(v['updates_per_s']),round(v['ms_per_pass'],2),v['pipelined'],v.get('pipeline_candidates_ms'))
PY
