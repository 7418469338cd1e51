mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chain_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/g41_chain -f python bench.py --config C2 --eta 0.9 --chunk 200 --no-extra --no-cpu --no-e2e --steps 1 --warmup 1 > gpurun_out/g41.log 2>&1; echo rc=$?
tail -c 300 gpurun_out/g41.log
