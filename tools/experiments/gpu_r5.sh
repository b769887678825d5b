for cfg in "16,4" "8,2" "4,2" "32,8" "0,0"; do
  TL_SYNC_DH=$cfg TL_SYNC_DW=$cfg timeout 200 ncu --clock-control none --kernel-name-base demangled --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:"EpiStore" -c 2 python tools/ncu_targets.py > gpurun_out/ncu_s.log 2>&1
  echo "SYNC $cfg"; grep -E "dram__bytes_read|duration" gpurun_out/ncu_s.log
done
