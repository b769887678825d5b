# dH / dW lockstep window probe (ncu DRAM bytes + serialised time), then a full capture of the step's GEMMs
p() { n=$1; shift
  env "$@" timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second -k regex:"gemm_sm100" -c 3 python tools/ncu_targets.py > gpurun_out/bw_$n.log 2>&1
  echo "== $n"; grep -E "gemm_sm100|dram__bytes|duration|per_second" gpurun_out/bw_$n.log | sed 's/(CUtensorMap_st.*//' | awk '{print "   ", $1, $2, $3, $4}'
}
p default
p dh81_dw81 TL_SYNC_DH=8,1 TL_SYNC_DW=8,1
p dh41_dw41 TL_SYNC_DH=4,1 TL_SYNC_DW=4,1
p dh161_dw161 TL_SYNC_DH=16,1 TL_SYNC_DW=16,1
p dh42_dw42 TL_SYNC_DH=4,2 TL_SYNC_DW=4,2
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_sm100|dsoftmax|pack_scatter|group_adv|traj_reduce|gather_rows" -c 10 -o gpurun_out/prof_r1b_full python tools/ncu_targets.py > gpurun_out/ncu_full_r1b.log 2>&1
tail -2 gpurun_out/ncu_full_r1b.log
ls -la gpurun_out/prof_r1b_full*
