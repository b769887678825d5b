# K3 branch-free templated token path: kernel times + ncu
set -x
timeout 600 python -m pytest tests/test_units_drop_gpu.py tests/test_gpu_parity.py -q -x -k "loss or pack or drop" --timeout=600 > gpurun_out/s2s_tests.log 2>&1; tail -2 gpurun_out/s2s_tests.log
timeout 300 python tools/kernel_times.py > gpurun_out/s2s_ktimes.log 2>&1; tail -1 gpurun_out/s2s_ktimes.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k[:40]:round(v['us'],1) for k,v in d['loss'].items() if k!='_span_us'})"
timeout 600 ncu --set full --clock-control none -k regex:"loss_unit" -c 1 -o gpurun_out/s2s_k3 python tools/ncu_membound.py > /dev/null 2>&1; ls gpurun_out/s2s_k3.ncu-rep
