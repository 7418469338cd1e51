mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_runner_modes.py -x -q --timeout=600 > gpurun_out/g31_tests.txt 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/g31_tests.txt
for ch in 50 200; do
timeout 600 python bench.py --config C2 --eta 0.9 --chunk $ch --no-extra --no-cpu --no-e2e > gpurun_out/g31_bench_$ch.json 2> gpurun_out/g31_bench_$ch.err; echo "bench rc=$?"; tail -3 gpurun_out/g31_bench_$ch.err
python - <<PY
import json
d=json.loads(open('gpurun_out/g31_bench_$ch.json').read().strip().splitlines()[-1])
print('chunk $ch value',d['value'],'ms',d['ms_per_step'],'pipelined',d.get('pipelined'))
print(d['stages_ms_per_step'])
for k,v in d['kernels'].items(): print(' ',k, round(v['ms_total_per_step'],3), v['launches_per_step'])
print(d['iters_hist'], d['method_counts'])
PY
done
