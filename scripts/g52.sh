for m in 0 128 160 192; do
echo "== LRZ_ARSVD_TAIL_MID=$m"
LRZ_ARSVD_TAIL_MID=$m python scripts/kprof_cfg.py C5 c128 20 64 3 2>&1 | tail -40 | sed -n 2,6p | grep -E "stages|tail"
done
