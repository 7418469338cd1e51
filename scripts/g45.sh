mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/g45_tests.txt 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/g45_tests.txt
for ch in 100 200; do
timeout 600 python bench.py --config C2 --eta 0.9 --chunk $ch --no-extra --no-cpu --no-e2e > gpurun_out/g33.json 2> gpurun_out/g33.err; echo "bench rc=$?"; tail -3 gpurun_out/g33.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g33.json').read().strip().splitlines()[-1])
print('chunk $ch value',round(d['value']),'ms',round(d['ms_per_step'],2), 'pipelined', d.get('pipelined'))
print({k:round(v,2) for k,v in d['stages_ms_per_step'].items()})
PY
done
python scripts/kprof_cfg.py C5 c128 20 64 3 2>&1 | tail -40 | head -14
