# default bench (as the driver runs it) + launch list of the headline
mkdir -p gpurun_out
start=$(date +%s)
timeout 1800 python bench.py > gpurun_out/g21_bench.json 2> gpurun_out/g21_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - start ))s"; tail -3 gpurun_out/g21_bench.err
