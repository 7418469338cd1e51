mkdir -p gpurun_out
for th in 64 128 256; do
LRZ_ARSVD_THREADS=$th LRZ_SCREEN_ROUNDS=16 timeout 600 python bench.py --config C2 --eta 0.9 --chunk 200 --no-extra --no-cpu --no-e2e > gpurun_out/g33.json 2> gpurun_out/g33.err; echo "bench rc=$?"; tail -3 gpurun_out/g33.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g33.json').read().strip().splitlines()[-1])
print('threads $th value',round(d['value']),'ms',round(d['ms_per_step'],2),'pipelined',d.get('pipelined'))
print({k:round(v,2) for k,v in d['stages_ms_per_step'].items()})
for k,v in d['kernels'].items():
    if k.startswith(('arsvd','sketch','chain','spec')): print(' ',k, round(v['ms_total_per_step'],3), v['launches_per_step'])
PY
done
