# Final evidence of the session: round-end script (tests, smoke, bench, launch
# list, ncu of two kernels), then the eta = 0.9 Woodbury-regime bench.
KERNELS="precode_dmma32 herm_inverse_warp" bash scripts/gpu_round.sh
timeout 300 python bench.py --eta 0.9 --no-graph --no-cpu --no-e2e --no-extra > gpurun_out/bench_eta09.json 2> gpurun_out/bench_eta09.err
echo "eta09 rc=$?"
