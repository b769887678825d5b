# A/B: dW red.add epilogue, fp16 logit stores evict_first, 2x chunk rows
timeout 600 python -m pytest tests -m gpu -q --timeout=180 -x > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
b() { # name, env..., args
  n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e $BARGS > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['step_frac'],4), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items()})" || tail -5 gpurun_out/bench_$n.log
}
b old TL_Z_POLICY=0 TL_DW_LOAD_ADD=1
b new TL_Z_POLICY=1 TL_DW_LOAD_ADD=0
b zonly TL_Z_POLICY=1 TL_DW_LOAD_ADD=1
BARGS="--chunk-rows 75776" b new2x TL_Z_POLICY=1 TL_DW_LOAD_ADD=0
for zp in 0 1; do
TL_Z_POLICY=$zp TL_DW_LOAD_ADD=$((1-zp)) timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second -k regex:"gemm_sm100" -c 3 python tools/ncu_targets.py > gpurun_out/ncu_dram_z$zp.log 2>&1
grep -E "gemm_sm100|dram__bytes|duration|per_second" gpurun_out/ncu_dram_z$zp.log | head -16
done
