# micro-batch parity + bench lines for the other BASELINE configs
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=300 -k "microbatch" > gpurun_out/t_r23.log 2>&1; tail -2 gpurun_out/t_r23.log
for c in c1 c5 c4 c3; do
  extra=""; [ $c = c3 ] && extra="--no-e2e"
  timeout 1500 python bench.py --config $c $extra > gpurun_out/bench_$c.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],1), round(d['value']), d['roofline'] and round(d['roofline']['frac'],4), d['roofline'] and round(d['roofline']['step_frac'],4), d['clocks']['sm_mhz'], d['config']['micro_batches'], d['config']['tokens_per_step'], d['report'])" || tail -5 gpurun_out/bench_$c.log
done
