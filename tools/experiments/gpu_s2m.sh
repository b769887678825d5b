# K1 scatter single-segment fast path; K3 fp32/int per-thread partials, 2-quad batches
set -x
timeout 900 python -m pytest tests/test_units_drop_gpu.py tests/test_gpu_parity.py tests/test_reference_dropin_gpu.py tests/test_determinism_gpu.py -q -x --timeout=600 > gpurun_out/s2m_tests.log 2>&1; tail -3 gpurun_out/s2m_tests.log
timeout 600 python tools/kernel_times.py > gpurun_out/s2m_ktimes.log 2>&1; tail -1 gpurun_out/s2m_ktimes.log
export MEMBOUND_ITERS=1
