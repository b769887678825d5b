# dW split-K tail: parity + A/B at C2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_determinism_gpu.py -m gpu -q --timeout=600 -x > gpurun_out/t_r41.log 2>&1; tail -3 gpurun_out/t_r41.log
grep -E "^E  " gpurun_out/t_r41.log | head -10
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if k.startswith('gemm')})" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b tail_$r
b notail_$r TL_DW_TAIL=0
done
