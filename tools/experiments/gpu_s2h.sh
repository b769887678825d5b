# ncu --set full of the K1 scatter / scan and the K3 streaming kernel at C2
set -x
export MEMBOUND_ITERS=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pack_scatter|pack_scan|loss_unit|loss_final" -c 4 -o gpurun_out/s2h_membound python tools/membound_bench.py > gpurun_out/s2h.log 2>&1; tail -3 gpurun_out/s2h.log; ls -la gpurun_out/s2h_membound.ncu-rep
