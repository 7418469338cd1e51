# Round-end evidence: GPU tests, smoke, default bench, launch list with per-kernel
# DRAM bytes, and ncu --set full captures of the top kernels (ncu runs only after
# the identical plain command exited 0).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout=400 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
ARGS="--steps 2 --warmup 1 --no-cpu --no-e2e --no-extra --no-graph"
if timeout 600 python bench.py $ARGS > gpurun_out/plain.log 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
      python bench.py $ARGS > gpurun_out/ncu_list.log 2>&1
  echo "list rc=$?"
  for k in ${KERNELS:-precode_dmma32 arsvd_screen sketch_cgemm gram_dmma herm_inverse_warp}; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
        -o gpurun_out/prof_$k -f python bench.py $ARGS > gpurun_out/ncu_$k.log 2>&1
    echo "$k rc=$?"
  done
fi
