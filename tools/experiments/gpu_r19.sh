# epilogue fast path + serpentine K + dH/dW window (16,1): tests, A/B bench, ncu DRAM/instr
timeout 600 python -m pytest tests -m gpu -q --timeout=180 -x > gpurun_out/t_r19.log 2>&1; tail -2 gpurun_out/t_r19.log
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e $BARGS > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['step_frac'],4), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items()})" || tail -5 gpurun_out/bench_$n.log
}
b new
b noserp TL_SERPENTINE=0
b oldwin TL_SYNC_DH=8,2 TL_SYNC_DW=8,2 TL_SERPENTINE=0
b new_again
for v in "new" "noserp TL_SERPENTINE=0"; do set -- $v; n=$1; shift
env "$@" timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:"gemm_sm100" -c 3 python tools/ncu_targets.py > gpurun_out/ncu19_$n.log 2>&1
echo "== $n"; grep -E "gemm_sm100|dram__bytes|duration|per_second|inst_exec|tensor" gpurun_out/ncu19_$n.log | sed 's/(CUtensorMap_st.*//' | awk '{print "   ", $1, $2, $3, $4}'
done
