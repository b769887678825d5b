# leaner dS pass: parity + bench A/B vs previous commit's numbers
timeout 900 python -m pytest tests -m gpu -q --timeout=600 -x > gpurun_out/t_r28.log 2>&1; tail -2 gpurun_out/t_r28.log
for i in 1 2; do
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_r28_$i.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_r28_$i.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['step_frac'],4), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items()})"
done
MEMBOUND_ITERS=5 timeout 600 python tools/membound_bench.py > gpurun_out/membound_r28.log 2>&1; tail -1 gpurun_out/membound_r28.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: v for k, v in d.items() if 'dsoftmax' in k})"
