# final verification after the K1 scan-tile change: full GPU suite + smoke, C2 bench, memory-bound kernels
set -x
rm -f gpurun_out/bwd_parity.jsonl gpurun_out/bwd_small_parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q --timeout=1500 > gpurun_out/s3p_tests.log 2>&1; tail -3 gpurun_out/s3p_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3p_smoke.log 2>&1; tail -1 gpurun_out/s3p_smoke.log
timeout 900 python bench.py > gpurun_out/s3p_bench_c2.log 2>&1; tail -1 gpurun_out/s3p_bench_c2.log | cut -c1-300
timeout 600 python tools/membound_bench.py > gpurun_out/s3p_membound.log 2>&1; tail -1 gpurun_out/s3p_membound.log | cut -c1-400
timeout 600 python tools/kernel_times.py > gpurun_out/s3p_ktimes.log 2>&1; tail -1 gpurun_out/s3p_ktimes.log | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pack_scan|pack_scatter|group_adv|loss_unit|loss_final" -o gpurun_out/s3p_membound python tools/ncu_membound.py > /dev/null 2>&1; ls -la gpurun_out/s3p_membound.ncu-rep
