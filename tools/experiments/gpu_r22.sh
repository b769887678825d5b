# round-1b evidence: tests, full bench line, launch list, ncu full capture, memory-bound kernels
timeout 900 python -m pytest tests -m gpu -q --timeout=300 > gpurun_out/t_r22.log 2>&1; tail -2 gpurun_out/t_r22.log
timeout 900 python bench.py > gpurun_out/bench_r22.log 2>&1; tail -1 gpurun_out/bench_r22.log | cut -c1-600
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r22.log 2>&1; tail -1 gpurun_out/bench_ref_r22.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile > gpurun_out/bench_ncu_r22.log 2>&1; wc -l gpurun_out/launches_r1b.csv
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_sm100|dsoftmax|pack_scatter|group_adv|traj_reduce|gather_rows" -c 10 -o gpurun_out/prof_r1b_full2 python tools/ncu_targets.py > gpurun_out/ncu_full_r22.log 2>&1; tail -1 gpurun_out/ncu_full_r22.log
timeout 600 python tools/membound_bench.py > gpurun_out/membound_r22.log 2>&1; tail -3 gpurun_out/membound_r22.log
