# ncu --set full captures of the DMMA Gram, fused precoder and warp inverse (C2 c128 probe)
set -x
mkdir -p gpurun_out
timeout 300 python scripts/dmma_probe.py > gpurun_out/probe.log 2>&1 || exit 1
for k in ${KERNELS:-gram_dmma precode_dmma32 herm_inverse_warp}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/prof_$k -f python scripts/dmma_probe.py > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
