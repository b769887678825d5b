timeout 600 python -m pytest tests -m gpu -q --timeout=180 > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
timeout 600 python tools/membound_bench.py > gpurun_out/membound.log 2>&1; tail -1 gpurun_out/membound.log
for k in pack_scatter pack_scan pack_padded group_adv loss32_traj dsoftmax gather_rows; do
MEMBOUND_ITERS=0 timeout 300 ncu --set full --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/mb_$k python tools/membound_bench.py > /dev/null 2>&1
done
ls gpurun_out/mb_*
