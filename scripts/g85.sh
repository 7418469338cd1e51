mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tensor_pipe.py tests/test_gpu_ops.py tests/test_gpu_configs_parity.py tests/test_gpu_fused_abi.py -x -q --timeout=900 2>&1 | tail -3
timeout 1200 python bench.py --no-cpu --no-e2e --no-extra --steps 3 --warmup 2 > gpurun_out/g85_bench.json 2> gpurun_out/g85_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/g85_bench.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g85_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline'], d['full_inverse']['ms_per_step'], d['mean_sum_rate'])
for k,v in list(d['kernels'].items())[:6]:
    print('  ',k, v['ms_total_per_step'], v.get('frac'))
PY
