mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/g14_bench.json 2> gpurun_out/g14_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/g14_ref.json 2> gpurun_out/g14_ref.err; echo "ref rc=$?"
python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g14_plain1.txt 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/g14_launch_C5c128.csv python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g14_ncu1.log 2>&1
echo "list rc=$?"
python scripts/prof_cfg.py C5 c64 20 > gpurun_out/g14_plain2.txt 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_w_kernel -s 2 -c 1 \
    -o gpurun_out/g14_tc_w_C5c64 -f python scripts/prof_cfg.py C5 c64 20 > gpurun_out/g14_ncu2.log 2>&1
echo "tc rc=$?"
