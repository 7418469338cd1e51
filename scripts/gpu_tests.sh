set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out; timeout 1200 python -m pytest tests -q -m gpu --timeout=400 --timeout-method=thread -x "$@" > gpurun_out/pytest_gpu.log 2>&1
tail -60 gpurun_out/pytest_gpu.log
