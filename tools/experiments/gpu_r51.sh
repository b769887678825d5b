# L2 hints round 2 (2 reps)
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if k.startswith('gemm')})" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b best_$r TL_DH_POLA=1 TL_DH_POLB=2 TL_DW_POLA=1 TL_DW_POLB=2
b wlast_$r TL_DH_POLB=2 TL_DW_POLB=2
b best_fwdwfirst_$r TL_DH_POLA=1 TL_DH_POLB=2 TL_DW_POLA=1 TL_DW_POLB=2 TL_FWD_POLB=1
done
