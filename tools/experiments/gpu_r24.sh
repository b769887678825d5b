timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=300 -k "microbatch" > gpurun_out/t_r24.log 2>&1; tail -2 gpurun_out/t_r24.log
bash tools/gpu_sanitize.sh
