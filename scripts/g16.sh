mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_tcgen05.py -q -x --timeout=240 > gpurun_out/g16_tc.txt 2>&1; echo "tc rc=$?"; tail -3 gpurun_out/g16_tc.txt
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --quick > gpurun_out/g10_bench.json 2> gpurun_out/g10_bench.err; echo "bench rc=$?"
timeout 1200 python -m pytest tests -q -m gpu -x --timeout=600 > gpurun_out/g10_pytest.txt 2>&1; tail -3 gpurun_out/g10_pytest.txt
