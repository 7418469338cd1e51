for m in 0 1; do
echo "== LRZ_ZGEMM_NARROW=$m"
LRZ_ZGEMM_NARROW=$m python scripts/kprof_cfg.py C4 c64 20 1024 3 2>&1 | tail -32 | grep -E "stages|chain|M_dmma|U_dmma|sketch"
LRZ_ZGEMM_NARROW=$m python scripts/kprof_cfg.py C5 c128 20 64 3 2>&1 | tail -32 | grep -E "stages"
done
timeout 1500 python -m pytest tests/test_gpu_configs_parity.py tests/test_gpu_tensor_pipe.py tests/test_gpu_fused_abi.py -x -q --timeout=900 2>&1 | tail -3
