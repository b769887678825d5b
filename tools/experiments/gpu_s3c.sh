# factored store at the benched shapes: full-shape backward parity (store / factored / recompute), full GPU suite, smoke
set -x
timeout 1800 python -m pytest tests/test_lmhead_bwd_fullshape_gpu.py -q -x --timeout=1500 > gpurun_out/s3c_fullshape.log 2>&1; tail -5 gpurun_out/s3c_fullshape.log
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -k "not full_shape_vs_oracle" > gpurun_out/s3c_tests.log 2>&1; tail -5 gpurun_out/s3c_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3c_smoke.log 2>&1; tail -2 gpurun_out/s3c_smoke.log
