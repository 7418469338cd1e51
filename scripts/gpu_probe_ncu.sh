# launch list of the arsvd probe (plain run first)
mkdir -p gpurun_out
python scripts/arsvd_probe.py 64 > gpurun_out/probe.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/probe_launches.csv \
    python scripts/arsvd_probe.py 64 > gpurun_out/probe_ncu.log 2>&1
echo rc=$?
cat gpurun_out/probe.log
