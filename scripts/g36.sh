mkdir -p gpurun_out
LRZ_SCREEN_ROUNDS=16 timeout 900 ncu --set full --import-source on --clock-control none -k regex:arsvd_small --launch-skip 2 --launch-count 1 -o gpurun_out/g36_arsvd_small -f python bench.py --config C2 --eta 0.9 --chunk 200 --no-extra --no-cpu --no-e2e --steps 1 --warmup 1 > gpurun_out/g36.log 2>&1; echo rc=$?
tail -3 gpurun_out/g36.log
