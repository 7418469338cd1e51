python scripts/probe_3m.py 2>&1 | head -8
for cfg in "128 1024 2560 c64" "64 1024 5120 c64" "100 500 320 c128" "288 1000 320 c128"; do set -- $cfg; for g3 in 0 1; do echo "== K=$1 N=$2 B=$3 $4 GRAM3M=$g3"; LRZ_GRAM3M=$g3 PK=$1 PN=$2 PB=$3 PDT=$4 python scripts/probe_3m.py 2>&1 | grep "gram\|G err"| head -5; done; done
timeout 900 python -m pytest tests/test_gpu_tensor_pipe.py tests/test_gpu_ops.py -x -q --timeout=600 2>&1 | tail -3
