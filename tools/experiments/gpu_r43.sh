# chunk size sweep (2 reps): 1x / 2x / 3x / 4x of 37888 action rows
b() { n=$1; shift
  timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-profile "$@" > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b c1x_$r
b c2x_$r --chunk-rows 75776
b c3x_$r --chunk-rows 113664
b c4x_$r --chunk-rows 151552
done
nvidia-smi --query-gpu=memory.total --format=csv
