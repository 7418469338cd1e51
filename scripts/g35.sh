mkdir -p gpurun_out
for cfg in "4 1" "6 1" "8 0" "6 0" "4 0"; do
set -- $cfg
LRZ_ARSVD_CTAS=$1 LRZ_ARSVD_SMEM=$2 LRZ_SCREEN_ROUNDS=16 timeout 600 python bench.py --config C2 --eta 0.9 --chunk 200 --no-extra --no-cpu --no-e2e > gpurun_out/g33.json 2> gpurun_out/g33.err; echo "bench rc=$?"; tail -3 gpurun_out/g33.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g33.json').read().strip().splitlines()[-1])
print('ctas $1 smem $2 value',round(d['value']),'ms',round(d['ms_per_step'],2))
for k,v in d['kernels'].items():
    if k.startswith(('arsvd_kernel')): print(' ',k, round(v['ms_total_per_step'],3), v['launches_per_step'])
PY
done
