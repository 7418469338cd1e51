mkdir -p gpurun_out
timeout 2400 python bench.py > gpurun_out/g47_bench.json 2> gpurun_out/g47_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/g47_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/g47_ref.json 2> gpurun_out/g47_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/g47_ref.json
