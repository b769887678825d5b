# output-store L2 hints for dH (dhidden) and dW (red.add) (2 reps) + parity of the hinted paths
timeout 900 env TL_DH_OUT_POLICY=1 TL_DW_OUT_POLICY=1 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=600 -x -k "lmhead_step or split_k or microbatch" > gpurun_out/t_r54.log 2>&1; tail -1 gpurun_out/t_r54.log
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if v > 100})" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b base_$r
b dhfirst_$r TL_DH_OUT_POLICY=1
b dwfirst_$r TL_DW_OUT_POLICY=1
b both_$r TL_DH_OUT_POLICY=1 TL_DW_OUT_POLICY=1
done
