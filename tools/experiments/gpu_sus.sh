timeout 400 python tools/sustained.py 24 > gpurun_out/sustained.log 2>&1
cat gpurun_out/sustained.log
