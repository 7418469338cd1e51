mkdir -p gpurun_out
timeout 1200 python bench.py --no-cpu --no-e2e --no-extra --steps 3 --warmup 2 > gpurun_out/g81_bench.json 2> gpurun_out/g81_bench.err; echo "bench rc=$?"; tail -5 gpurun_out/g81_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/g81_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['pipelined'], d['pipeline_candidates_ms'], d['roofline']['frac'], d['full_inverse'])
PY
timeout 900 python -m pytest tests/test_gpu_trajectory.py -x -q --timeout=600 2>&1 | tail -3
