# ncu --set full of the memory-bound kernels at C2 (second launch of each); compute-sanitizer on the current kernels
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pack_scan|pack_scatter|group_adv|loss_unit|loss_final" -o gpurun_out/s2r_membound python tools/ncu_membound.py > gpurun_out/s2r_ncu.log 2>&1; tail -2 gpurun_out/s2r_ncu.log; ls -la gpurun_out/s2r_membound.ncu-rep
bash tools/gpu_sanitize.sh > gpurun_out/s2r_sanitize.log 2>&1; cat gpurun_out/s2r_sanitize.log
