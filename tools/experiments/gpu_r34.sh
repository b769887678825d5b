# dH/dW epilogue: double-buffered TMEM slices vs one at a time (A/B builds), + parity
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_determinism_gpu.py -m gpu -q --timeout=600 -x > gpurun_out/t_r34.log 2>&1; tail -2 gpurun_out/t_r34.log
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if k.startswith('gemm')})" || tail -5 gpurun_out/bench_$n.log
}
for r in 1 2; do
b pipe_$r
TL_EXTRA_NVCC_FLAGS="-DTL_EPI_PIPELINE=0" python -c "from paper_2509_01055_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
b serial_$r
python -c "from paper_2509_01055_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
done
