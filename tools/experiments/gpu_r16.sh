# forward GEMM wave-shape / L2 policy probe: DRAM bytes (ncu) + event timing
v() { n=$1; shift
  env "$@" timeout 120 python tools/fwd_probe.py 2>&1 | tail -1 | sed "s/^/$n /"
  env "$@" PROBE_ITERS=0 timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read.sum -k regex:gemm_sm100 -s 1 -c 1 python tools/fwd_probe.py > gpurun_out/probe_$n.log 2>&1
  grep -E "dram__bytes|duration|per_second|lts__t" gpurun_out/probe_$n.log | awk '{print "   ", $1, $2, $3}'
}
v default
v pola0 TL_FWD_POLA=0
v pola1 TL_FWD_POLA=1
v nosync TL_SYNC_FWD=0,0
v win1 TL_SYNC_FWD=56,1
v strips2 TL_FWD_STRIPS=2
v strips12 TL_FWD_STRIPS=12
v gm74 TL_FWD_GROUPM=74
v gm2s37 TL_FWD_GROUPM=2 TL_FWD_STRIPS=37
