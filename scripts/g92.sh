for m in 0 1; do
for dt in c128 c64; do
LRZ_GRAM32_3M=$m timeout 600 python bench.py --config C2 --dtype $dt --no-cpu --no-e2e --no-extra --steps 10 --warmup 3 > gpurun_out/g92_$m$dt.json 2> gpurun_out/g92_$m$dt.err || tail -3 gpurun_out/g92_$m$dt.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g92_$m$dt.json').read().strip().splitlines()[-1])
k=d['kernels'].get('gram_dmma_kernel',{})
print('GRAM32_3M=$m $dt', round(d['value']), round(d['ms_per_step'],3), 'full', round(d['full_inverse']['ms_per_step'],3), 'gram ms', round(k.get('ms_total_per_step',0),3), d['mean_sum_rate'])
PY
done; done
python -m pytest tests/test_gpu_tensor_pipe.py tests/test_gpu_ops.py tests/test_gpu_trajectory.py -x -q 2>&1 | tail -2
