mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_trajectory.py tests/test_gpu_runner_modes.py -x -q --timeout=600 > gpurun_out/g34_tests.txt 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/g34_tests.txt
bash scripts/g33.sh
