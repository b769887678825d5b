# round 2: ncu DRAM counters of the memory-bound kernels (K1/K2/K3 + reductions) at C2
set -x
export MEMBOUND_ITERS=2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none --csv --log-file gpurun_out/s2b_membound_ncu.csv -k regex:"pack_|group_adv|loss32|traj_reduce|group_reduce|report_kernel|dsoftmax|gather" python tools/membound_bench.py > gpurun_out/s2b_membound.log 2>&1; tail -1 gpurun_out/s2b_membound.log | cut -c1-300
timeout 600 python tools/membound_bench.py > gpurun_out/s2b_membound_timed.log 2>&1; tail -1 gpurun_out/s2b_membound_timed.log
