set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout=120 -k "not gemm and not lmhead" 2>&1 | tail -30 > gpurun_out/t_small.log
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=60 -k "gemm" 2>&1 | tail -40 > gpurun_out/t_gemm.log
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=90 -k "lmhead" 2>&1 | tail -40 > gpurun_out/t_lmhead.log
timeout 120 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
cat gpurun_out/t_small.log gpurun_out/t_gemm.log gpurun_out/t_lmhead.log gpurun_out/smoke.log | tail -80
