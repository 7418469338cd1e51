mkdir -p gpurun_out
for cfg in "C3 c64 50" "C5 c64 20"; do set -- $cfg
python scripts/prof_cfg.py $1 $2 $3 > gpurun_out/g95_plain_$1$2.txt 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/g95_launch_$1$2.csv python scripts/prof_cfg.py $1 $2 $3 > gpurun_out/g95_ncu_$1$2.log 2>&1
echo "list $1 $2 rc=$?"
done
