set -x
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=120 -x 2>&1 | tail -25 > gpurun_out/t_all.log
cat gpurun_out/t_all.log
timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1
cat gpurun_out/gemm_bench.log
timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1
cat gpurun_out/bench_c2.log
