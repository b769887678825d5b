# coarser lockstep steps: forward 4 / 8 tiles, dH/dW 64 / 128 / 256 k-blocks (2 reps, interleaved)
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-profile > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b A_f224_b64_$r TL_SYNC_FWD=224,1 TL_SYNC_DH=64,1 TL_SYNC_DW=64,1
b B_f448_b64_$r TL_SYNC_FWD=448,1 TL_SYNC_DH=64,1 TL_SYNC_DW=64,1
b C_f224_b128_$r TL_SYNC_FWD=224,1 TL_SYNC_DH=128,1 TL_SYNC_DW=128,1
b D_f448_b128_$r TL_SYNC_FWD=448,1 TL_SYNC_DH=128,1 TL_SYNC_DW=128,1
b E_f224_b256_$r TL_SYNC_FWD=224,1 TL_SYNC_DH=256,1 TL_SYNC_DW=256,1
done
