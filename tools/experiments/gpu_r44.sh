# adaptive chunk (up to 4 x 37888 rows): tests + C2 bench + C5 (largest activations) + C3 micro-batched
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 -x > gpurun_out/t_r44.log 2>&1; tail -2 gpurun_out/t_r44.log
for c in c2 c5 c3; do
  timeout 1800 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/bench_r44_$c.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_r44_$c.log').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],1), round(d['value']), d['config']['chunk_rows'], d['config'].get('micro_batches'), round(d['roofline']['frac'],4), round(d['roofline']['step_frac'],4), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_r44_$c.log
done
nvidia-smi --query-gpu=memory.used --format=csv
