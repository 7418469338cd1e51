mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_cond_guard.py -q -x --timeout=500 > gpurun_out/g17_ops.txt 2>&1; echo "ops rc=$?"; tail -3 gpurun_out/g17_ops.txt
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --quick > gpurun_out/g10_bench.json 2> gpurun_out/g10_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/g10_bench.err
timeout 1200 python -m pytest tests -q -m gpu -x --timeout=600 > gpurun_out/g10_pytest.txt 2>&1; tail -3 gpurun_out/g10_pytest.txt
