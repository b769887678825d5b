# lockstep granularity A/B with serpentine on; 7-stage ring for 256-wide tiles
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['step_frac'],4), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if k.startswith('gemm')})" || tail -5 gpurun_out/bench_$n.log
}
b A_default
b B_fwd_nosync TL_SYNC_FWD=0,0
b C_fwd_14_4 TL_SYNC_FWD=14,4
b D_fwd_28_2 TL_SYNC_FWD=28,2
b E_bwd_nosync TL_SYNC_DH=0,0 TL_SYNC_DW=0,0
b F_bwd_8_2 TL_SYNC_DH=8,2 TL_SYNC_DW=8,2
TL_STAGES256=7 python -c "from paper_2509_01055_b200 import _build; _build.build(force=True)" 2>&1 | tail -1
b G_stages7
b H_stages7_14_4 TL_SYNC_FWD=14,4
python -c "from paper_2509_01055_b200 import _build; _build.build(force=True)" 2>&1 | tail -1
b A_default_again
