timeout 600 python -m pytest tests -m gpu -q --timeout=180 -x > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
timeout 900 python bench.py --config c2 --steps 2 --warmup 3 > gpurun_out/bench_c2.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_c2.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['step_frac'], d['clocks'], d['kernel_ms_per_step'], d['cpu_baseline']['value'])"
