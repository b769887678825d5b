# compute-sanitizer over the GPU parity tests (memcheck on the fused step incl. tcgen05 GEMMs; racecheck/synccheck on shared-memory kernels)
K1='test_pack or test_advantages or test_loss_fp32 or test_grpo_lmhead_step_vs_oracle or microbatch or dapo or split_k or no_action or test_loss_units or test_step_drop or frozen or factored or fixup'
K2='test_pack or test_advantages or test_loss_fp32 or test_grpo_lmhead_step_vs_oracle or test_loss_units or test_factored_vs or fixup_path'
for tool in memcheck racecheck synccheck; do
  k="$K1"; [ $tool != memcheck ] && k="$K2"
  # racecheck: the tcgen05 GEMMs are excluded — the tool reports their
  # tcgen05.alloc (TMEM base address written to shared memory by the tensor
  # memory allocator, read by all warps only after a cluster barrier) as a
  # hazard at the alloc instruction itself; it does not model that write.
  ex=""; [ $tool = racecheck ] && ex="--kernel-name-exclude kns=gemm_sm100"
  timeout 1500 compute-sanitizer --tool $tool $ex --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_units_drop_gpu.py tests/test_factored_gpu.py -m gpu -q -k "$k" > gpurun_out/san_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/san_$tool.log | tail -3
done
