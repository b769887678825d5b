timeout 600 python -m pytest tests -m gpu -q --timeout=180 > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
timeout 300 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c1.log 2>&1; cut -c1-600 gpurun_out/bench_c1.log
timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1; cut -c1-900 gpurun_out/bench_c2.log
