# dH / dW lockstep step under the final L2 priorities (2 reps)
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-profile > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b base_$r
b b32_$r TL_SYNC_DH=32,1 TL_SYNC_DW=32,1
b b128_$r TL_SYNC_DH=128,1 TL_SYNC_DW=128,1
done
