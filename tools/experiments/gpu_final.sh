# end-of-round evidence on the final tree -> gpurun_out/final4_* (copied into profiles/ by hand)
set -x
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 > gpurun_out/final4_tests.log 2>&1; tail -2 gpurun_out/final4_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4_smoke.log 2>&1; tail -1 gpurun_out/final4_smoke.log
timeout 900 python bench.py > gpurun_out/final4_bench_c2.log 2>&1; tail -1 gpurun_out/final4_bench_c2.log | cut -c1-200
timeout 600 python bench.py --impl reference > gpurun_out/final4_bench_ref.log 2>&1; tail -1 gpurun_out/final4_bench_ref.log | cut -c1-200
for c in c1 c5 c4; do timeout 1500 python bench.py --config $c > gpurun_out/final4_bench_$c.log 2>&1; tail -1 gpurun_out/final4_bench_$c.log | cut -c1-120; done
timeout 1800 python bench.py --config c3 --no-e2e > gpurun_out/final4_bench_c3.log 2>&1; tail -1 gpurun_out/final4_bench_c3.log | cut -c1-120
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final4_launches_c2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile > /dev/null 2>&1; wc -l gpurun_out/final4_launches_c2.csv
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_sm100|dsoftmax|pack_scatter|group_adv|traj_reduce|gather_rows" -c 10 -o gpurun_out/final4_full python tools/ncu_targets.py > /dev/null 2>&1; ls -la gpurun_out/final4_full.ncu-rep
timeout 600 python tools/membound_bench.py > gpurun_out/final4_membound.log 2>&1; tail -1 gpurun_out/final4_membound.log | cut -c1-200
