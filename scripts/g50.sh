timeout 1500 python -m pytest tests/test_gpu_configs_parity.py tests/test_gpu_tensor_pipe.py tests/test_gpu_fused_abi.py tests/test_gpu_trajectory.py tests/test_gpu_cond_guard.py -x -q --timeout=900 2>&1 | tail -5
python scripts/kprof_cfg.py C3 c64 50 256 3 2>&1 | tail -32 | head -10
