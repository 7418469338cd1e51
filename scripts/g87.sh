mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/g87_tests.txt 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/g87_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
( time timeout 2400 python bench.py > gpurun_out/g87_bench.json 2> gpurun_out/g87_bench.err ) 2>&1 | tail -3; echo "bench rc=$?"; tail -3 gpurun_out/g87_bench.err
python scripts/bench_summary.py gpurun_out/g87_bench.json 2>&1 | tail -40
