set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=60 -k "gemm" 2>&1 | tail -5 > gpurun_out/t_gemm.log
timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1
timeout 400 python bench.py --config c2s --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c2s.log 2>&1
timeout 600 python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/bench_c2.log 2>&1
cat gpurun_out/t_gemm.log gpurun_out/gemm_bench.log gpurun_out/bench_c2s.log gpurun_out/bench_c2.log | tail -60
