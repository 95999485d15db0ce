# compute-sanitizer over tools/sanitize_step.py (logs -> gpurun_out/)
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --target-processes all python tools/sanitize_step.py \
      > gpurun_out/${SAN_PREFIX:-r2}_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/${SAN_PREFIX:-r2}_sanitizer_$tool.log
done
