mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tensor_pipe.py tests/test_gpu_ops.py -x -q --timeout=600 2>&1 | tail -3
for m3 in 1 0; do
LRZ_3M=$m3 timeout 1200 python bench.py --no-cpu --no-e2e --no-extra --steps 3 --warmup 2 > gpurun_out/g84_bench_$m3.json 2> gpurun_out/g84_bench_$m3.err; echo "bench rc=$?"; tail -3 gpurun_out/g84_bench_$m3.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g84_bench_$m3.json').read().strip().splitlines()[-1])
print('3M=$m3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['full_inverse']['ms_per_step'], d['mean_sum_rate'])
for k in ('w_dmma_direct_kernel','gram_dmma_off_kernel','coupling_dmma_direct'):
    print('  ',k, d['kernels'][k]['ms_total_per_step'], d['kernels'][k].get('frac'))
PY
done
