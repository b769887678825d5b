# experiment: anchored log-sum-exp in the factored forward epilogue (no running max, q = e) vs current; C2 A/B on one box
set -x
TOOLLOOP_B200_LIB=paper_2509_01055_b200/_objs/anch/libtoolloop_b200.so timeout 600 python -m pytest tests/test_factored_gpu.py -q -x -k "vs_fp16 and 256" > gpurun_out/s3m_tests.log 2>&1; tail -3 gpurun_out/s3m_tests.log
for i in 1 2; do
  for v in base anch; do
    if [ $v = base ]; then unset TOOLLOOP_B200_LIB; else export TOOLLOOP_B200_LIB=paper_2509_01055_b200/_objs/$v/libtoolloop_b200.so; fi
    timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/s3m_bench_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3m_bench_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k:round(x,1) for k,x in d['kernel_ms_per_step'].items() if x>1})"
  done
done
