mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_tcgen05.py -q -x --timeout=240 > gpurun_out/g8_tc.txt 2>&1
echo "rc=$?"; tail -30 gpurun_out/g8_tc.txt
