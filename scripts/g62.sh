mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/g62_tests.txt 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/g62_tests.txt
timeout 2400 python bench.py > gpurun_out/g62_bench.json 2> gpurun_out/g62_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/g62_bench.err
python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g62_plain1.txt 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/g62_launch_C5c128.csv python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g62_ncu1.log 2>&1
echo "list C5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:w_dmma_direct -s 1 -c 1 \
    -o gpurun_out/g62_w_direct_C5c128 -f python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g62_ncu2.log 2>&1
echo "w rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_dmma_off -s 1 -c 1 \
    -o gpurun_out/g62_gram_off_C5c128 -f python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g62_ncu3.log 2>&1
echo "gram rc=$?"
