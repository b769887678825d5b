# tightened LM-head tolerances; full-shape sampled-row parity; store vs recompute at C2 shape
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=600 -k "lmhead or full_shape" > gpurun_out/t_r27.log 2>&1; tail -3 gpurun_out/t_r27.log
grep -E "^E  " gpurun_out/t_r27.log | head -20
