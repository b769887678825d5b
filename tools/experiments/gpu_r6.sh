timeout 900 python bench.py --config c2 --steps 2 --warmup 3 > gpurun_out/bench_c2.log 2>&1
cat gpurun_out/bench_c2.log
