mkdir -p gpurun_out
for extra in "" "--no-coresident"; do
timeout 1200 python bench.py --no-cpu --no-e2e --no-extra --steps 3 --warmup 2 --pipe heavy $extra > gpurun_out/g83_bench.json 2> gpurun_out/g83_bench.err; echo "bench rc=$?"; tail -5 gpurun_out/g83_bench.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/g83_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['pipelined'], d['pipeline_candidates_ms'], d['roofline']['frac'], d['full_inverse']['ms_per_step'])
PY
done
