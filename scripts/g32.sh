mkdir -p gpurun_out
for cfg in "200 16" "200 32" "200 64" "50 8" "50 16" "50 32"; do
set -- $cfg
LRZ_SCREEN_ROUNDS=$2 timeout 600 python bench.py --config C2 --eta 0.9 --chunk $1 --no-extra --no-cpu --no-e2e > gpurun_out/g32.json 2> gpurun_out/g32.err; echo "bench rc=$?"; tail -3 gpurun_out/g32.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g32.json').read().strip().splitlines()[-1])
print('chunk $1 rounds $2 value',round(d['value']),'ms',round(d['ms_per_step'],2),'pipelined',d.get('pipelined'))
print({k:round(v,2) for k,v in d['stages_ms_per_step'].items()})
for k,v in d['kernels'].items():
    if k.startswith(('arsvd','sketch','chain','spec')): print(' ',k, round(v['ms_total_per_step'],3), v['launches_per_step'])
PY
done
