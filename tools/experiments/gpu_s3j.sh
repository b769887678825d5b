# full GPU suite (incl. the new K1 tests on the scan + scatter path and C1 full-shape parity) + smoke
set -x
rm -f gpurun_out/bwd_parity.jsonl gpurun_out/bwd_small_parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q --timeout=1500 > gpurun_out/s3j_tests.log 2>&1; tail -4 gpurun_out/s3j_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3j_smoke.log 2>&1; tail -1 gpurun_out/s3j_smoke.log
