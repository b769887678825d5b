# GEMM stall accounting (profiling build on the box)
TL_GEMM_STATS=1 python -c "from paper_2509_01055_b200 import _build; _build.build(force=True)" 2>&1 | tail -1
timeout 300 python tools/gemm_stats.py 2>&1 | tail -5
TL_SYNC_FWD=0,0 TL_SYNC_DH=0,0 TL_SYNC_DW=0,0 timeout 300 python tools/gemm_stats.py 2>&1 | tail -3
