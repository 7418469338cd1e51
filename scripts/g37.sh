mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_trajectory.py tests/test_gpu_runner_modes.py tests/test_gpu_leo.py -x -q --timeout=600 > gpurun_out/g37_tests.txt 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/g37_tests.txt
for pc in 0 1; do
LRZ_ARSVD_PRECOND=$pc LRZ_SCREEN_ROUNDS=16 timeout 600 python bench.py --config C2 --eta 0.9 --chunk 200 --no-extra --no-cpu --no-e2e > gpurun_out/g33.json 2> gpurun_out/g33.err; echo "bench rc=$?"; tail -3 gpurun_out/g33.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g33.json').read().strip().splitlines()[-1])
print('precond $pc value',round(d['value']),'ms',round(d['ms_per_step'],2))
for k,v in d['kernels'].items():
    if k.startswith(('arsvd_kernel')): print(' ',k, round(v['ms_total_per_step'],3), v['launches_per_step'])
PY
done
