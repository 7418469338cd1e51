mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/g30_tests.txt 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/g30_tests.txt
timeout 1500 python bench.py > gpurun_out/g30_bench.json 2> gpurun_out/g30_bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/g30_bench.json; tail -5 gpurun_out/g30_bench.err
