# round 2: bench lines for the other configs on the new K1 / K3 kernels
set -x
for c in c1 c5 c4; do timeout 1500 python bench.py --config $c > gpurun_out/s2o_bench_$c.log 2>&1; tail -1 gpurun_out/s2o_bench_$c.log | cut -c1-300; done
timeout 1800 python bench.py --config c3 --no-e2e > gpurun_out/s2o_bench_c3.log 2>&1; tail -1 gpurun_out/s2o_bench_c3.log | cut -c1-300
for c in c5 c1; do timeout 300 python tools/kernel_times.py $c > gpurun_out/s2o_ktimes_$c.log 2>&1; tail -1 gpurun_out/s2o_ktimes_$c.log | cut -c1-200; done
