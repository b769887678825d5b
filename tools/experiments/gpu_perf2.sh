set -x
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=120 -x 2>&1 | tail -15 > gpurun_out/t_all.log
timeout 120 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --config c2 --steps 2 --warmup 3 > gpurun_out/bench_c2.log 2>&1
timeout 300 python bench.py --impl reference --config c2 --steps 1 --warmup 1 > gpurun_out/bench_ref.log 2>&1
nproc > gpurun_out/host.txt; free -g >> gpurun_out/host.txt; lscpu | head -20 >> gpurun_out/host.txt
cat gpurun_out/t_all.log gpurun_out/smoke.log gpurun_out/bench_c2.log gpurun_out/bench_ref.log gpurun_out/host.txt | tail -60
