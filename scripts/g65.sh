python scripts/kprof_cfg.py C4 c64 20 1024 3 2>&1 | tail -32 | grep -E "stages|coupling"
python scripts/kprof_cfg.py C3 c64 50 256 3 2>&1 | tail -32 | grep -E "stages|coupling"
python scripts/kprof_cfg.py C5 c128 20 64 3 2>&1 | tail -32 | grep -E "stages|coupling|w_dmma"
