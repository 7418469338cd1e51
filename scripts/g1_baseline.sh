mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
lscpu | head -20 > gpurun_out/g1_cpu.txt; nproc >> gpurun_out/g1_cpu.txt; free -g >> gpurun_out/g1_cpu.txt
timeout 300 python scripts/stage_probe_cfg.py C5 25 c128 > gpurun_out/g1_stage.txt 2>&1
timeout 300 python scripts/stage_probe_cfg.py C5 25 c64 >> gpurun_out/g1_stage.txt 2>&1
timeout 300 python scripts/stage_probe_cfg.py C3 50 c64 >> gpurun_out/g1_stage.txt 2>&1
timeout 300 python scripts/stage_probe_cfg.py C4 20 c64 >> gpurun_out/g1_stage.txt 2>&1
timeout 300 python scripts/stage_probe_cfg.py C2 200 c128 0.9 >> gpurun_out/g1_stage.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -x --timeout=400 > gpurun_out/g1_pytest.txt 2>&1
tail -3 gpurun_out/g1_pytest.txt
