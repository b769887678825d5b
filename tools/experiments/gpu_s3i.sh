# K1 single-pass packer, scatter unrolled x4: tiles of 16 (base) / 8 / 32 segments vs scan + scatter (pack2k)
set -x
timeout 900 python -m pytest tests/test_units_drop_gpu.py tests/test_gpu_parity.py -q -x --timeout=600 -k "pack or drop or flatten" > gpurun_out/s3i_tests.log 2>&1; tail -3 gpurun_out/s3i_tests.log
for i in 1 2; do
  for v in base t8 t32 pack2k; do
    if [ $v = base ]; then unset TOOLLOOP_B200_LIB; else export TOOLLOOP_B200_LIB=paper_2509_01055_b200/_objs/$v/libtoolloop_b200.so; fi
    timeout 300 python tools/kernel_times.py > gpurun_out/s3i_kt_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3i_kt_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, 'pack', {k[-24:]:round(v['us'],1) for k,v in d['pack'].items() if k!='_span_us'})"
    MEMBOUND_ITERS=20 timeout 600 python tools/membound_bench.py > gpurun_out/s3i_mb_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3i_mb_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, {k[:30]:(v['ms'],v['frac_of_hbm']) for k,v in d.items() if isinstance(v,dict) and ('K1' in k)})"
  done
done
unset TOOLLOOP_B200_LIB
for c in c5 c1 c3; do timeout 300 python tools/kernel_times.py $c > gpurun_out/s3i_kt_$c.log 2>&1; tail -1 gpurun_out/s3i_kt_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', {k[-24:]:round(v['us'],1) for k,v in d['pack'].items() if k!='_span_us'})"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pack_fused" -c 1 -o gpurun_out/s3i_k1 python tools/ncu_membound.py > /dev/null 2>&1; ls gpurun_out/s3i_k1.ncu-rep
