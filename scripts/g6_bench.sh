mkdir -p gpurun_out
( time timeout 1500 python bench.py --steps 2 --warmup 1 --quick ) > gpurun_out/g6_bench.json 2> gpurun_out/g6_bench.err
echo "bench rc=$?"
tail -5 gpurun_out/g6_bench.err
( time timeout 600 python bench.py --impl reference --steps 2 --warmup 1 ) > gpurun_out/g6_ref.json 2> gpurun_out/g6_ref.err
echo "ref rc=$?"; tail -3 gpurun_out/g6_ref.err
