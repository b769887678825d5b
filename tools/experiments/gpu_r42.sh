# env A/Bs on the final tree: L2 hints, chunk size (2 reps, interleaved)
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-profile $BARGS > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b base_$r
b zpol0_$r TL_Z_POLICY=0
b pola0_$r TL_FWD_POLA=0
BARGS="--chunk-rows 75776" b chunk2x_$r
done
