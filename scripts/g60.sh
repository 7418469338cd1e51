timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_tensor_pipe.py -x -q --timeout=600 2>&1 | tail -3
for m in 1 0; do
echo "== LRZ_GRAM_DIAG=$m"
LRZ_GRAM_DIAG=$m python scripts/kprof_cfg.py C3 c64 50 256 3 2>&1 | tail -32 | grep -E "gram"
LRZ_GRAM_DIAG=$m python scripts/kprof_cfg.py C4 c64 20 1024 3 2>&1 | tail -32 | grep -E "gram"
LRZ_GRAM_DIAG=$m python scripts/kprof_cfg.py C5 c128 20 64 3 2>&1 | tail -32 | grep -E "gram"
LRZ_GRAM_DIAG=$m python scripts/kprof_cfg.py C5 c64 20 64 3 2>&1 | tail -32 | grep -E "gram"
done
