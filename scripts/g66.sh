nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
for m in 1 0 1; do
echo "== LRZ_W_DIRECT=$m"
LRZ_W_DIRECT=$m python scripts/kprof_cfg.py C5 c128 20 64 3 2>&1 | tail -32 | grep -E "w_dmma|:W |coupling|gram_dmma"
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active --format=csv
