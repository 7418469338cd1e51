mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_configs_parity.py tests/test_gpu_trajectory.py tests/test_gpu_fused_abi.py -x -q --timeout=900 > gpurun_out/g46_tests.txt 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/g46_tests.txt
python scripts/kprof_cfg.py C5 c128 20 64 3 2>&1 | tail -40 | head -10
python scripts/kprof_cfg.py C4 c64 20 1024 3 2>&1 | tail -32 | head -10
python scripts/kprof_cfg.py C3 c64 50 256 3 2>&1 | tail -32 | head -12
