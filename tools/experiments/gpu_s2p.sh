# round 2 evidence on the current tree: full GPU suite, smoke, C2 bench, memory-bound kernels,
# ncu launch list of the C2 bench command, ncu --set full of one ~1-chunk step
set -x
rm -f gpurun_out/bwd_small_parity.jsonl gpurun_out/bwd_parity.jsonl
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -rs > gpurun_out/s2p_tests.log 2>&1; tail -3 gpurun_out/s2p_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2p_smoke.log 2>&1; tail -1 gpurun_out/s2p_smoke.log
timeout 900 python bench.py > gpurun_out/s2p_bench_c2.log 2>&1; tail -1 gpurun_out/s2p_bench_c2.log | cut -c1-300
timeout 600 python tools/membound_bench.py > gpurun_out/s2p_membound.log 2>&1; tail -1 gpurun_out/s2p_membound.log | cut -c1-200
timeout 600 python tools/kernel_times.py > gpurun_out/s2p_ktimes.log 2>&1; tail -1 gpurun_out/s2p_ktimes.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2p_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile > /dev/null 2>&1; wc -l gpurun_out/s2p_launches_c2.csv
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_sm100|dsoftmax|pack_scatter|pack_scan|group_adv|loss_unit|loss_final|gather_rows" -c 12 -o gpurun_out/s2p_full python tools/ncu_targets.py > /dev/null 2>&1; ls -la gpurun_out/s2p_full.ncu-rep
