# forward shape knobs on the final tree: strips, ring depth (2 reps)
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-profile > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b base_$r
b strips12_$r TL_FWD_STRIPS=12
b strips2_$r TL_FWD_STRIPS=2
TL_STAGES256=7 python -c "from paper_2509_01055_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
b stages7_$r
python -c "from paper_2509_01055_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
done
