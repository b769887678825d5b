# round 2: new K1 (look-back scan + PDL scatter, drop bits), K3 token-parallel units, step options
set -x
timeout 900 python -m pytest tests/test_units_drop_gpu.py tests/test_gpu_parity.py -q -x --timeout=600 > gpurun_out/s2c_tests.log 2>&1; tail -25 gpurun_out/s2c_tests.log
timeout 600 python tools/membound_bench.py > gpurun_out/s2c_membound.log 2>&1; tail -1 gpurun_out/s2c_membound.log
export MEMBOUND_ITERS=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/s2c_membound_ncu.csv -k regex:"pack_|group_adv|loss_unit" -c 12 python tools/membound_bench.py > /dev/null 2>&1; wc -l gpurun_out/s2c_membound_ncu.csv
