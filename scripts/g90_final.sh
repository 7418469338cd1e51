mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/g90_tests.txt 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/g90_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
( time timeout 2400 python bench.py > gpurun_out/g90_bench.json 2> gpurun_out/g90_bench.err ) 2>&1 | tail -3; echo "bench rc=$?"; tail -3 gpurun_out/g90_bench.err
( time timeout 900 python bench.py --impl reference > gpurun_out/g90_ref.json 2> gpurun_out/g90_ref.err ) 2>&1 | tail -3; echo "ref rc=$?"
python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g90_plain2.txt 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/g90_launch_C2eta09.csv python scripts/prof_cfg.py C2 c128 200 64 0.9 > gpurun_out/g90_ncu2.log 2>&1
echo "list C2 rc=$?"
