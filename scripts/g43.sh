python scripts/kprof_cfg.py C5 c128 20 64 3 2>&1 | tail -40
python scripts/kprof_cfg.py C4 c64 20 1024 3 2>&1 | tail -32
