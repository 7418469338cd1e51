mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rng.py tests/test_gpu_leo.py -q -x --timeout=500 > gpurun_out/g22_rng.txt 2>&1; echo "rng rc=$?"; tail -4 gpurun_out/g22_rng.txt
