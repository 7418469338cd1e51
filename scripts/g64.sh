for m in 1 0; do
echo "== LRZ_SKETCH_DIRECT=$m"
LRZ_SKETCH_DIRECT=$m python scripts/kprof_cfg.py C5 c128 20 64 3 2>&1 | tail -32 | grep -E "stages|sketch"
LRZ_SKETCH_DIRECT=$m python scripts/kprof_cfg.py C4 c64 20 1024 3 2>&1 | tail -32 | grep -E "stages|sketch"
LRZ_SKETCH_DIRECT=$m python scripts/kprof_cfg.py C3 c64 50 256 3 2>&1 | tail -32 | grep -E "stages|sketch"
done
timeout 1500 python -m pytest tests/test_gpu_configs_parity.py tests/test_gpu_tensor_pipe.py tests/test_gpu_ops.py tests/test_gpu_fused_abi.py -x -q --timeout=900 2>&1 | tail -3
