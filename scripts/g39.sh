mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ops.py tests/test_gpu_trajectory.py tests/test_gpu_runner_modes.py tests/test_gpu_leo.py tests/test_gpu_tensor_pipe.py tests/test_gpu_cond_guard.py tests/test_gpu_fused_abi.py -x -q --timeout=600 > gpurun_out/g39_tests.txt 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/g39_tests.txt
for ch in 200 50; do
timeout 600 python bench.py --config C2 --eta 0.9 --chunk $ch --no-extra --no-cpu --no-e2e > gpurun_out/g33.json 2> gpurun_out/g33.err; echo "bench rc=$?"; tail -3 gpurun_out/g33.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g33.json').read().strip().splitlines()[-1])
print('chunk $ch value',round(d['value']),'ms',round(d['ms_per_step'],2))
print({k:round(v,2) for k,v in d['stages_ms_per_step'].items()})
for k,v in d['kernels'].items():
    if k.startswith(('arsvd','chain','sketch')): print(' ',k, round(v['ms_total_per_step'],3), v['launches_per_step'])
PY
done
