# K3 warp walker (TL_K3_WALK=1, units of 1,024 tokens) vs CTA walker (k3cta build): tests + kernel times + device times
set -x
timeout 900 python -m pytest tests/test_units_drop_gpu.py tests/test_gpu_parity.py tests/test_determinism_gpu.py tests/test_dp_equality_gpu.py tests/test_reference_dropin_gpu.py -q -x --timeout=600 > gpurun_out/s3e_tests.log 2>&1; tail -3 gpurun_out/s3e_tests.log
for i in 1 2; do
  for v in base k3cta; do
    if [ $v = base ]; then unset TOOLLOOP_B200_LIB; else export TOOLLOOP_B200_LIB=paper_2509_01055_b200/_objs/$v/libtoolloop_b200.so; fi
    timeout 300 python tools/kernel_times.py > gpurun_out/s3e_kt_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3e_kt_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, {k[:30]:round(v['us'],1) for k,v in d['loss'].items() if k!='_span_us'}, 'span', round(d['loss']['_span_us'],1))"
    timeout 600 python tools/membound_bench.py > gpurun_out/s3e_mb_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3e_mb_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, {k[:40]:(v['ms'],v['frac_of_hbm']) for k,v in d.items() if isinstance(v,dict)})"
  done
done
unset TOOLLOOP_B200_LIB
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"loss_unit" -c 1 -o gpurun_out/s3e_k3 python tools/ncu_membound.py > /dev/null 2>&1; ls gpurun_out/s3e_k3.ncu-rep
