# new defaults (fwd 2-tile steps, dH/dW 32) vs coarser; + full GPU suite on the refactored lmhead
timeout 900 python -m pytest tests -m gpu -q --timeout=600 -x > gpurun_out/t_r31.log 2>&1; tail -2 gpurun_out/t_r31.log
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-profile > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b new_$r
b old_$r TL_SYNC_FWD=56,1 TL_SYNC_DH=16,1 TL_SYNC_DW=16,1
b coarse_$r TL_SYNC_FWD=224,1 TL_SYNC_DH=64,1 TL_SYNC_DW=64,1
done
