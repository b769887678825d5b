# final-tree evidence: full GPU suite + smoke, every config, reference arm, memory-bound kernels, ncu launch list + full capture
set -x
rm -f gpurun_out/bwd_parity.jsonl gpurun_out/bwd_small_parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q --timeout=1500 > gpurun_out/s3l_tests.log 2>&1; tail -3 gpurun_out/s3l_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3l_smoke.log 2>&1; tail -1 gpurun_out/s3l_smoke.log
timeout 900 python bench.py > gpurun_out/s3l_bench_c2.log 2>&1; tail -1 gpurun_out/s3l_bench_c2.log | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/s3l_bench_ref.log 2>&1; tail -1 gpurun_out/s3l_bench_ref.log | cut -c1-200
for c in c1 c5 c4; do timeout 1500 python bench.py --config $c > gpurun_out/s3l_bench_$c.log 2>&1; tail -1 gpurun_out/s3l_bench_$c.log | cut -c1-200; done
timeout 1800 python bench.py --config c3 --no-e2e > gpurun_out/s3l_bench_c3.log 2>&1; tail -1 gpurun_out/s3l_bench_c3.log | cut -c1-200
timeout 600 python tools/membound_bench.py > gpurun_out/s3l_membound.log 2>&1; tail -1 gpurun_out/s3l_membound.log | cut -c1-300
timeout 600 python tools/kernel_times.py > gpurun_out/s3l_ktimes.log 2>&1; tail -1 gpurun_out/s3l_ktimes.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3l_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile > /dev/null 2>&1; wc -l gpurun_out/s3l_launches_c2.csv
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_sm100|dsoftmax|pack_scatter|pack_scan|group_adv|loss_unit|loss_final|gather_rows|gather_anchor|fixup_rows|scale_rows" -c 14 -o gpurun_out/s3l_full python tools/ncu_targets.py > /dev/null 2>&1; ls -la gpurun_out/s3l_full.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pack_scan|pack_scatter|group_adv|loss_unit|loss_final" -o gpurun_out/s3l_membound python tools/ncu_membound.py > /dev/null 2>&1; ls -la gpurun_out/s3l_membound.ncu-rep
