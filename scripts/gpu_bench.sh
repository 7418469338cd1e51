# GPU round trip: tests, smoke, bench, launch list (ncu only after the plain run exits 0)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout=400 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
