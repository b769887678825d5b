set -x
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=120 2>&1 | tail -4
timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"gemm_sm100" -c 3 python tools/ncu_targets.py > gpurun_out/ncu_dram.log 2>&1
grep -E "gemm_sm100|dram__bytes|duration" gpurun_out/ncu_dram.log | head -30
timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c2.log 2>&1
cat gpurun_out/bench_c2.log
