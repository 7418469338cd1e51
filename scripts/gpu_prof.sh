# tests + bench + ncu evidence (ncu only after the identical plain command exited 0)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout=400 --timeout-method=thread > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
ARGS="--steps 2 --warmup 1 --no-cpu --no-e2e --no-extra"
if [ "${PROFILE:-1}" = "1" ]; then
  timeout 600 python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_list.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-arsvd} -s 2 -c 1 \
      -o gpurun_out/prof_${KNAME:-arsvd} -f python bench.py $ARGS > gpurun_out/ncu_full.log 2>&1
  echo "ncu rc=$?"
fi
