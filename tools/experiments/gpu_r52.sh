# new L2-priority defaults: tests, bench confirm, ncu DRAM per GEMM
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 -x > gpurun_out/t_r52.log 2>&1; tail -2 gpurun_out/t_r52.log
for r in 1 2; do
timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_r52_$r.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_r52_$r.log').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['step_frac'],4), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if v > 1})"
done
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:"gemm_sm100" -c 3 python tools/ncu_targets.py > gpurun_out/ncu_r52.log 2>&1
grep -E "gemm_sm100|dram__bytes|duration|tensor" gpurun_out/ncu_r52.log | sed 's/(CUtensorMap_st.*//' | awk '{print "   ", $1, $2, $3, $4}'
