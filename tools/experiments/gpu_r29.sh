# vectorised K3: parity + ncu bandwidth of the memory-bound kernels at C2
timeout 900 python -m pytest tests -m gpu -q --timeout=600 -x > gpurun_out/t_r29.log 2>&1; tail -2 gpurun_out/t_r29.log
for k in pack_scatter pack_scan pack_padded group_adv loss32_traj dsoftmax gather_rows; do
MEMBOUND_ITERS=0 timeout 300 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:$k -s 1 -c 1 python tools/membound_bench.py > gpurun_out/mb29_$k.log 2>&1
echo "== $k"; grep -E "dram__bytes|duration" gpurun_out/mb29_$k.log | awk '{print "   ", $1, $2, $3}'
done
