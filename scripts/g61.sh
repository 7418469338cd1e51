for m in 1 2; do
echo "== LRZ_W_NBW=$m"
LRZ_W_NBW=$m python scripts/kprof_cfg.py C5 c128 20 64 3 2>&1 | tail -32 | grep -E "w_dmma"
done
