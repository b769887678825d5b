set -x
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"gemm_sm100|nvjet|dsoftmax|pack_scatter|group_adv|traj_reduce|gather_rows|combine" -c 14 -o gpurun_out/prof_r1 python tools/ncu_targets.py > gpurun_out/ncu_full.log 2>&1
tail -5 gpurun_out/ncu_full.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 1 --no-cpu --no-e2e --no-profile > gpurun_out/bench_c2_ncu.log 2>&1
tail -2 gpurun_out/bench_c2_ncu.log; wc -l gpurun_out/launches_c2.csv
ls -la gpurun_out
