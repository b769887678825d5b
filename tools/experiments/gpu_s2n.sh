# K3 grid shape A/B: persistent (4 CTAs/SM) vs 1 / 2 / 4 slots per CTA
set -x
for v in base k3s1 k3s2 k3s4; do
  if [ $v = base ]; then unset TOOLLOOP_B200_LIB; else export TOOLLOOP_B200_LIB=paper_2509_01055_b200/_objs/$v/libtoolloop_b200.so; fi
  timeout 300 python tools/kernel_times.py > gpurun_out/s2n_$v.log 2>&1; tail -1 gpurun_out/s2n_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', {k[:30]:round(v['us'],1) for k,v in d['loss'].items() if k!='_span_us'})"
done
