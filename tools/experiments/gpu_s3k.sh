# K3 occupancy: 4 CTAs/SM x 2-quad batches (base) vs 5 / 6 CTAs, 6 / 8 CTAs x 1-quad batches
set -x
for i in 1 2; do
  for v in base c5 c6 c6b1 c8b1; do
    if [ $v = base ]; then unset TOOLLOOP_B200_LIB; else export TOOLLOOP_B200_LIB=paper_2509_01055_b200/_objs/$v/libtoolloop_b200.so; fi
    timeout 300 python tools/kernel_times.py > gpurun_out/s3k_kt_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3k_kt_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, 'loss', {k[-24:]:round(v['us'],1) for k,v in d['loss'].items() if k!='_span_us'})"
    MEMBOUND_ITERS=20 timeout 600 python tools/membound_bench.py > gpurun_out/s3k_mb_${v}_$i.log 2>&1
    tail -1 gpurun_out/s3k_mb_${v}_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', $i, {k[:30]:(v['ms'],v['frac_of_hbm']) for k,v in d.items() if isinstance(v,dict) and ('K3' in k)})"
  done
done
