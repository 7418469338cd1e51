# round-2 evidence after the 3M kernels: launch list (time + DRAM) of the headline
# workload, full ncu captures of the 3M W kernel (C5 c128) and the 3M Gram (C5 c64)
mkdir -p gpurun_out
python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g88_plain1.txt 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/g88_launch_C5c128.csv python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g88_ncu1.log 2>&1
echo "list C5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:w_dmma_3m_tiled -s 1 -c 1 \
    -o gpurun_out/g88_w3m_C5c128 -f python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g88_ncu2.log 2>&1
echo "w3m rc=$?"
python scripts/prof_cfg.py C5 c64 20 > gpurun_out/g88_plain3.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_dmma_3m_tiled -s 1 -c 1 \
    -o gpurun_out/g88_gram3m_C5c64 -f python scripts/prof_cfg.py C5 c64 20 > gpurun_out/g88_ncu3.log 2>&1
echo "gram3m rc=$?"
tail -1 gpurun_out/g88_plain*.txt
