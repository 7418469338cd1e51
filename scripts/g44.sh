mkdir -p gpurun_out
for cfg in "96 8 200" "96 6 200" "64 8 200" "128 6 100" "128 6 200"; do
set -- $cfg
LRZ_ARSVD_THREADS=$1 LRZ_ARSVD_CTAS=$2 timeout 600 python bench.py --config C2 --eta 0.9 --chunk $3 --no-extra --no-cpu --no-e2e > gpurun_out/g33.json 2> gpurun_out/g33.err; echo "bench rc=$?"; tail -3 gpurun_out/g33.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g33.json').read().strip().splitlines()[-1])
print('threads $1 ctas $2 chunk $3 value',round(d['value']),'ms',round(d['ms_per_step'],2), 'pipelined', d.get('pipelined'))
print({k:round(v,2) for k,v in d['stages_ms_per_step'].items()})
PY
done
