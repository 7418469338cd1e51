# state check after the container re-creation: GPU tests, smoke, default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu --timeout=600 > gpurun_out/g20_pytest.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/g20_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g20_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/g20_smoke.log
/usr/bin/time -v timeout 1800 python bench.py > gpurun_out/g20_bench.json 2> gpurun_out/g20_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/g20_bench.err
timeout 1200 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g20_ref.json 2> gpurun_out/g20_ref.err; echo "ref rc=$?"
