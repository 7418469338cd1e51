mkdir -p gpurun_out
timeout 300 python scripts/stage_probe_cfg.py C5 25 c128 > gpurun_out/g4_stage.txt 2>&1
timeout 300 python scripts/stage_probe_cfg.py C3 50 c64 >> gpurun_out/g4_stage.txt 2>&1
timeout 300 python scripts/stage_probe_cfg.py C4 20 c64 >> gpurun_out/g4_stage.txt 2>&1
timeout 300 python scripts/stage_probe_cfg.py C2 200 c128 >> gpurun_out/g4_stage.txt 2>&1
cat gpurun_out/g4_stage.txt
timeout 900 python -m pytest tests -q -m gpu -x --timeout=600 > gpurun_out/g4_pytest.txt 2>&1
tail -5 gpurun_out/g4_pytest.txt
