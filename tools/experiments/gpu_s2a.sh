# round 2: verify the tree after the full-shape parity / NCCL commit
set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -rs > gpurun_out/s2a_tests.log 2>&1; tail -15 gpurun_out/s2a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a_smoke.log 2>&1; tail -2 gpurun_out/s2a_smoke.log
timeout 900 python bench.py > gpurun_out/s2a_bench_c2.log 2>&1; tail -1 gpurun_out/s2a_bench_c2.log | cut -c1-400
timeout 900 python bench.py --impl reference > gpurun_out/s2a_bench_ref.log 2>&1; tail -1 gpurun_out/s2a_bench_ref.log | cut -c1-400
