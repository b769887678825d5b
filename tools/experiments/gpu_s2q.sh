# A/B on one box: packed fp32x2 epilogue / dS pass (default) vs scalar (nof2); K1 warp look-back; K3 fp64 fused-step partials
set -x
timeout 900 python -m pytest tests/test_dp_equality_gpu.py tests/test_units_drop_gpu.py tests/test_determinism_gpu.py tests/test_gpu_parity.py -q -x --timeout=600 > gpurun_out/s2q_tests.log 2>&1; tail -3 gpurun_out/s2q_tests.log
timeout 300 python tools/kernel_times.py > gpurun_out/s2q_ktimes.log 2>&1; tail -1 gpurun_out/s2q_ktimes.log | cut -c1-600
for i in 1 2; do
  for v in base nof2; do
    if [ $v = base ]; then unset TOOLLOOP_B200_LIB; else export TOOLLOOP_B200_LIB=paper_2509_01055_b200/_objs/$v/libtoolloop_b200.so; fi
    timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/s2q_bench_${v}_$i.log 2>&1
    tail -1 gpurun_out/s2q_bench_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k:round(x,1) for k,x in d['kernel_ms_per_step'].items() if x>1})"
  done
done
