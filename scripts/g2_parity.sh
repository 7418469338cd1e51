mkdir -p gpurun_out
rm -f gpurun_out/parity_*.json
timeout 1500 python -m pytest tests/test_gpu_configs_parity.py -q -s --timeout=1400 > gpurun_out/g2_parity.txt 2>&1
tail -40 gpurun_out/g2_parity.txt
