mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/g71_tests.txt 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/g71_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 2400 python bench.py > gpurun_out/g71_bench.json 2> gpurun_out/g71_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/g71_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/g71_ref.json 2> gpurun_out/g71_ref.err; echo "ref rc=$?"
python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g71_plain1.txt 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/g71_launch_C5c128.csv python scripts/prof_cfg.py C5 c128 20 > gpurun_out/g71_ncu1.log 2>&1
echo "list C5 rc=$?"
python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g71_plain2.txt 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/g71_launch_C2eta09.csv python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g71_ncu2.log 2>&1
echo "list C2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 0 -c 1 \
    -o gpurun_out/g71_chain_C2eta09 -f python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g71_ncu3.log 2>&1
echo "chain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_kernel -s 1 -c 1 \
    -o gpurun_out/g71_chain_C3 -f python scripts/prof_cfg.py C3 c64 50 > gpurun_out/g71_ncu4.log 2>&1
echo "chain C3 rc=$?"
