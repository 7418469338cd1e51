# round-2 final evidence: launch lists (time + DRAM) of the headline workload and of
# C2 eta 0.9, full ncu captures of the new kernels (each command first run plain)
mkdir -p gpurun_out
python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g53_plain1.txt 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/g53_launch_C5c128.csv python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g53_ncu1.log 2>&1
echo "list C5 rc=$?"
python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g53_plain2.txt 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/g53_launch_C2eta09.csv python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g53_ncu2.log 2>&1
echo "list C2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 \
    -o gpurun_out/g53_chain_C2eta09 -f python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g53_ncu3.log 2>&1
echo "chain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:arsvd_small -s 1 -c 1 \
    -o gpurun_out/g53_arsvd_small_C2eta09 -f python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g53_ncu4.log 2>&1
echo "arsvd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:arsvd_screen -s 3 -c 1 \
    -o gpurun_out/g53_screen_C2eta09 -f python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g53_ncu5.log 2>&1
echo "screen rc=$?"
python scripts/prof_cfg.py C3 c64 50 > gpurun_out/g53_plain3.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 \
    -o gpurun_out/g53_chain_C3 -f python scripts/prof_cfg.py C3 c64 50 > gpurun_out/g53_ncu6.log 2>&1
echo "chain C3 rc=$?"
tail -2 gpurun_out/g53_plain*.txt
