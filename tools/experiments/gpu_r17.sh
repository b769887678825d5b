# pipelined-mode tests + A/B bench; forward lockstep window probe with DRAM bytes
timeout 600 python -m pytest tests/test_determinism_gpu.py tests/test_gpu_parity.py -m gpu -q --timeout=180 -x > gpurun_out/t_r17.log 2>&1; tail -2 gpurun_out/t_r17.log
b() { n=$1; shift
  env "$@" timeout 900 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e $BARGS > gpurun_out/bench_$n.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$n.log').read().strip().splitlines()[-1]); print('$n', round(d['ms_per_step'],1), round(d['value']), round(d['roofline']['frac'],4), round(d['roofline']['step_frac'],4), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in d['kernel_ms_per_step'].items()})" || tail -5 gpurun_out/bench_$n.log
}
BARGS="--mode store" b store
BARGS="--mode pipelined" b pipe
BARGS="--mode store" b store_win1 TL_SYNC_FWD=56,1
BARGS="--mode pipelined" b pipe_win1 TL_SYNC_FWD=56,1
v() { n=$1; shift
  env "$@" PROBE_ITERS=10 timeout 120 python tools/fwd_probe.py 2>&1 | tail -1 | sed "s/^/$n /"
  env "$@" PROBE_ITERS=1 timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second -k regex:gemm_sm100 -s 1 -c 1 python tools/fwd_probe.py > gpurun_out/probe_$n.log 2>&1
  grep -E "dram__bytes|duration|per_second" gpurun_out/probe_$n.log | awk '{print "   ", $1, $2, $3}'
}
v default
v win1 TL_SYNC_FWD=56,1
v half1 TL_SYNC_FWD=28,1
v half2 TL_SYNC_FWD=28,2
v win1s2 TL_SYNC_FWD=56,1 TL_FWD_STRIPS=2
v default_again
