# K3 finalize: unit rows loaded 4 at a time (base) vs one at a time (fin0)
set -x
timeout 600 python -m pytest tests/test_units_drop_gpu.py tests/test_gpu_parity.py tests/test_dp_equality_gpu.py tests/test_determinism_gpu.py -q -x > gpurun_out/s3q_tests.log 2>&1; tail -1 gpurun_out/s3q_tests.log
for i in 1 2; do
  for v in base fin0; do
    if [ $v = base ]; then unset TOOLLOOP_B200_LIB; else export TOOLLOOP_B200_LIB=paper_2509_01055_b200/_objs/$v/libtoolloop_b200.so; fi
    timeout 300 python tools/kernel_times.py > gpurun_out/s3q_kt_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3q_kt_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, 'loss', {k[-24:]:round(v['us'],1) for k,v in d['loss'].items() if k!='_span_us'})"
    MEMBOUND_ITERS=20 timeout 600 python tools/membound_bench.py > gpurun_out/s3q_mb_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3q_mb_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, {k[:30]:(v['ms'],v['frac_of_hbm']) for k,v in d.items() if isinstance(v,dict) and ('K3' in k)})"
  done
done
