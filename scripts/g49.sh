for m in 65 64; do
echo "== LRZ_INV_BLOCKED_MIN=$m"
LRZ_INV_BLOCKED_MIN=$m python scripts/kprof_cfg.py C3 c64 50 256 3 conv 2>&1 | tail -12 | head -9
done
LRZ_INV_BLOCKED_MIN=64 timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_cond_guard.py tests/test_gpu_configs_parity.py -x -q --timeout=900 -k "inverse or cond or C3" 2>&1 | tail -3
