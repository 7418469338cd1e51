mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:w_dmma_3m_tiled -s 2 -c 1 \
    -o gpurun_out/g89_w3m_C5c128 -f python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g89_ncu1.log 2>&1
echo "w3m rc=$?"
LRZ_GRAM3M=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_dmma_3m_tiled -s 1 -c 1 \
    -o gpurun_out/g89_gram3m_C5c128 -f python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g89_ncu2.log 2>&1
echo "gram3m c128 rc=$?"
