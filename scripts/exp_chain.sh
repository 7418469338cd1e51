# A/B of the resident chain at the headline config (chain stage ms)
for v in "LRZ_CHAIN_RESIDENT=1" "LRZ_CHAIN_RESIDENT=0" "LRZ_CHAIN_CARVEOUT=100" "LRZ_CHAIN_CARVEOUT=0"; do
  env $v timeout 200 python bench.py --steps 10 --no-cpu --no-e2e --no-extra > gpurun_out/ec.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ec.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), round(d['stages']['chain']['ms'],4), round(d['stages']['precode_rate']['ms'],4))" >> gpurun_out/ec_summary.txt
done
