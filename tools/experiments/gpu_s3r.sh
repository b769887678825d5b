# steady state (10 timed steps) and the backward modes on the final tree, C2, one box
set -x
timeout 1200 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/s3r_bench_10steps.log 2>&1; tail -1 gpurun_out/s3r_bench_10steps.log | cut -c1-300
for m in store-fp16 recompute; do timeout 1200 python bench.py --no-cpu --no-e2e --mode $m > gpurun_out/s3r_bench_$m.log 2>&1; tail -1 gpurun_out/s3r_bench_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], d['roofline']['frac'], d['roofline']['issued_frac'])"; done
