mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 0 -c 1 \
    -o gpurun_out/g53_chain_C2eta09 -f python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g53_ncu3.log 2>&1
echo "chain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:arsvd_small -s 0 -c 1 \
    -o gpurun_out/g53_arsvd_small_C2eta09 -f python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g53_ncu4.log 2>&1
echo "arsvd rc=$?"
