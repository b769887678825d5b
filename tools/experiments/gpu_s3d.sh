# round-2 evidence after the factored backward: C2 bench (+ reference arm), other configs,
# memory-bound kernels (clean-L2 flush), ncu launch list of the C2 bench, ncu --set full of a 1-chunk step
set -x
timeout 900 python bench.py > gpurun_out/s3d_bench_c2.log 2>&1; tail -1 gpurun_out/s3d_bench_c2.log | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/s3d_bench_ref.log 2>&1; tail -1 gpurun_out/s3d_bench_ref.log | cut -c1-300
for c in c1 c5 c4; do timeout 1500 python bench.py --config $c > gpurun_out/s3d_bench_$c.log 2>&1; tail -1 gpurun_out/s3d_bench_$c.log | cut -c1-200; done
timeout 1800 python bench.py --config c3 --no-e2e > gpurun_out/s3d_bench_c3.log 2>&1; tail -1 gpurun_out/s3d_bench_c3.log | cut -c1-200
timeout 600 python tools/membound_bench.py > gpurun_out/s3d_membound.log 2>&1; tail -1 gpurun_out/s3d_membound.log | cut -c1-300
MEMBOUND_FLUSH=write timeout 600 python tools/membound_bench.py > gpurun_out/s3d_membound_wflush.log 2>&1; tail -1 gpurun_out/s3d_membound_wflush.log | cut -c1-300
timeout 600 python tools/kernel_times.py > gpurun_out/s3d_ktimes.log 2>&1; tail -1 gpurun_out/s3d_ktimes.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3d_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile > /dev/null 2>&1; wc -l gpurun_out/s3d_launches_c2.csv
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_sm100|dsoftmax|pack_scatter|pack_scan|group_adv|loss_unit|loss_final|gather_rows|gather_anchor|fixup_rows|scale_rows" -c 14 -o gpurun_out/s3d_full python tools/ncu_targets.py > /dev/null 2>&1; ls -la gpurun_out/s3d_full.ncu-rep
