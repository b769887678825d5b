timeout 600 python -m pytest tests -m gpu -q --timeout=180 > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
timeout 600 python tools/cli_bench.py 32 > gpurun_out/cli_bench.log 2>&1; tail -3 gpurun_out/cli_bench.log
