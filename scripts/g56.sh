for m in 0 128 96; do
echo "== LRZ_ARSVD_P1_SMALL=$m"
LRZ_ARSVD_P1_SMALL=$m python scripts/kprof_cfg.py C3 c64 50 256 3 2>&1 | tail -30 | grep -E "arsvd_kernel|stages"
LRZ_ARSVD_P1_SMALL=$m python scripts/kprof_cfg.py C4 c64 20 1024 3 2>&1 | tail -30 | grep -E "arsvd_kernel|stages"
done
