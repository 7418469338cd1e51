mkdir -p gpurun_out
python scripts/prof_cfg.py C5 c128 25 > gpurun_out/g5_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:arsvd_kernel -s 1 -c 1 \
   -o gpurun_out/g5_arsvd_C5 -f python scripts/prof_cfg.py C5 c128 25 > gpurun_out/g5_ncu.log 2>&1
echo rc=$?
tail -3 gpurun_out/g5_ncu.log
