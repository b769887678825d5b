timeout 600 python -m pytest tests -m gpu -q --timeout=180 > gpurun_out/t_all.log 2>&1; tail -15 gpurun_out/t_all.log
