for c in 0 2 1; do for p in 0 -1; do
  LRZ_GRAM_CTAS_PER_SM=$c LRZ_RNG_PRIO=$p timeout 200 python bench.py --steps 10 --no-cpu --no-e2e --no-extra > gpurun_out/exp_${c}_${p}.json 2> gpurun_out/exp_${c}_${p}.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/exp_${c}_${p}.json').read().strip().splitlines()[-1]); print('cap=$c prio=$p', round(d['ms_per_step'],4), round(d['value']), d['stages']['gram']['ms'])" >> gpurun_out/exp_summary.txt 2>&1
done; done
