# lockstep window A/B with serpentine + per-strip forward lockstep (2 reps each, interleaved)
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-profile > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b base_$r
b fwd56_2_$r TL_SYNC_FWD=56,2
b fwd112_1_$r TL_SYNC_FWD=112,1
b bwd32_1_$r TL_SYNC_DH=32,1 TL_SYNC_DW=32,1
done
