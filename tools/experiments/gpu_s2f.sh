# round 2: persistent K3 units, merged K1 scatter searches; device timing behind a spin kernel
set -x
timeout 900 python -m pytest tests/test_units_drop_gpu.py tests/test_gpu_parity.py tests/test_reference_dropin_gpu.py tests/test_determinism_gpu.py -q -x --timeout=600 > gpurun_out/s2f_tests.log 2>&1; tail -5 gpurun_out/s2f_tests.log
timeout 600 python tools/membound_bench.py > gpurun_out/s2f_membound.log 2>&1; tail -1 gpurun_out/s2f_membound.log
timeout 600 python tools/kernel_times.py > gpurun_out/s2f_ktimes.log 2>&1; tail -1 gpurun_out/s2f_ktimes.log
