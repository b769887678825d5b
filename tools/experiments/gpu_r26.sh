# full GPU suite + smoke (driver's round-end checks) on the current tree
timeout 900 python -m pytest tests -m gpu -q --timeout=300 > gpurun_out/t_r26.log 2>&1; tail -2 gpurun_out/t_r26.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r26.log 2>&1; python -c "import json; d=json.loads(open('gpurun_out/bench_r26.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],1), round(d['value']), d['e2e']['value'], d['roofline']['frac'], d['roofline']['step_frac'], d['roofline']['traffic'], d['clocks'], d['gpu_launches'])"
