# round 2 (session 3) start: verify the restored tree — full GPU suite, smoke, C2 bench
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -rs > gpurun_out/s3a_tests.log 2>&1; tail -15 gpurun_out/s3a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3a_smoke.log 2>&1; tail -2 gpurun_out/s3a_smoke.log
timeout 900 python bench.py --no-cpu > gpurun_out/s3a_bench_c2.log 2>&1; tail -1 gpurun_out/s3a_bench_c2.log | cut -c1-600
