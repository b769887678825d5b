# sanitizers on the current kernels; backward-mode comparison at C2
bash tools/gpu_sanitize.sh
for m in recompute pipelined store; do
  timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --mode $m > gpurun_out/bench_mode_$m.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_mode_$m.log').read().strip().splitlines()[-1]); print('$m', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['step_frac'],4), round(d['roofline']['issued_frac'],4), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if v > 1})"
done
