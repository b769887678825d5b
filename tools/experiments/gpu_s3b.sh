# factored store (bf16 q, no dS pass): new tests + step suites; C2 A/B factored vs fp16 store on one box
set -x
timeout 900 python -m pytest tests/test_factored_gpu.py -q -x --timeout=600 > gpurun_out/s3b_factored.log 2>&1; tail -15 gpurun_out/s3b_factored.log
timeout 1200 python -m pytest tests -m gpu -q --timeout=900 -k "not fullshape" > gpurun_out/s3b_tests.log 2>&1; tail -15 gpurun_out/s3b_tests.log
for i in 1 2; do
  for m in store store-fp16; do
    timeout 900 python bench.py --no-cpu --no-e2e --mode $m > gpurun_out/s3b_bench_${m}_$i.log 2>&1
    tail -1 gpurun_out/s3b_bench_${m}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', $i, round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k:round(x,1) for k,x in d['kernel_ms_per_step'].items() if x>1})"
  done
done
