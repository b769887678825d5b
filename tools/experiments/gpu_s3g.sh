# N2 overlap test + full GPU suite + smoke on the current tree; C2 bench; sanitizers incl. the factored kernels
set -x
timeout 1800 python -m pytest tests -m gpu -q --timeout=900 > gpurun_out/s3g_tests.log 2>&1; tail -4 gpurun_out/s3g_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3g_smoke.log 2>&1; tail -1 gpurun_out/s3g_smoke.log
timeout 900 python bench.py > gpurun_out/s3g_bench_c2.log 2>&1; tail -1 gpurun_out/s3g_bench_c2.log | cut -c1-250
bash tools/gpu_sanitize.sh > gpurun_out/s3g_sanitize.log 2>&1; cat gpurun_out/s3g_sanitize.log
