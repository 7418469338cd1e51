mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 \
    -o gpurun_out/g70_chain_C3 -f python scripts/prof_cfg.py C3 c64 50 > gpurun_out/g70.log 2>&1
echo rc=$?
