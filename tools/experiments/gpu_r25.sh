timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=300 -k "microbatch" > gpurun_out/t_r25.log 2>&1; tail -2 gpurun_out/t_r25.log
bash tools/gpu_sanitize.sh
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['step_frac'],4), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if k.startswith('gemm')})" || tail -5 gpurun_out/bench_$n.log
}
b base
b split TL_SYNC_SPLIT_FWD=1
b base2
b split2 TL_SYNC_SPLIT_FWD=1
