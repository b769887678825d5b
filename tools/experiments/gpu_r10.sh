timeout 300 python -m pytest tests/test_determinism_gpu.py -q 2>&1 | tail -1
timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --chunk-rows 75776 > gpurun_out/bench_c2_big.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_c2_big.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['clocks'], d['kernel_ms_per_step'])"
