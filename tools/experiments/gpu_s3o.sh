# K1 scatter shape: 256 threads x 4 rounds unrolled 2 (base) vs unroll 4, 128 x 8, 512 x 2, 256 x 2
set -x
for v in u4 t128 t512 r2; do TOOLLOOP_B200_LIB=paper_2509_01055_b200/_objs/$v/libtoolloop_b200.so timeout 600 python -m pytest tests/test_units_drop_gpu.py tests/test_gpu_parity.py -q -x -k "pack" > gpurun_out/s3o_tests_$v.log 2>&1; tail -1 gpurun_out/s3o_tests_$v.log; done
for i in 1 2; do
  for v in base u4 t128 t512 r2; do
    if [ $v = base ]; then unset TOOLLOOP_B200_LIB; else export TOOLLOOP_B200_LIB=paper_2509_01055_b200/_objs/$v/libtoolloop_b200.so; fi
    timeout 300 python tools/kernel_times.py > gpurun_out/s3o_kt_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3o_kt_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, 'pack', {k[-24:]:round(v['us'],1) for k,v in d['pack'].items() if k!='_span_us'})"
    MEMBOUND_ITERS=20 timeout 600 python tools/membound_bench.py > gpurun_out/s3o_mb_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3o_mb_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, {k[:30]:(v['ms'],v['frac_of_hbm']) for k,v in d.items() if isinstance(v,dict) and ('K1' in k)})"
  done
done
