mkdir -p gpurun_out
for cfg in "6 1 50" "6 0 50" "8 0 50" "6 0 25" "6 0 100"; do
set -- $cfg
LRZ_ARSVD_CTAS=$1 LRZ_ARSVD_SMEM=$2 timeout 600 python bench.py --config C2 --eta 0.9 --chunk $3 --no-extra --no-cpu --no-e2e > gpurun_out/g33.json 2> gpurun_out/g33.err; echo "bench rc=$?"; tail -3 gpurun_out/g33.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g33.json').read().strip().splitlines()[-1])
print('ctas $1 smem $2 chunk $3 value',round(d['value']),'ms',round(d['ms_per_step'],2), 'pipelined', d.get('pipelined'))
print({k:round(v,2) for k,v in d['stages_ms_per_step'].items()})
PY
done
