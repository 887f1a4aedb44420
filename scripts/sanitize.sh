#!/bin/bash
# compute-sanitizer over the engine (VERDICT r01 "Robustness"): memcheck on every kernel test,
# and memcheck / racecheck / synccheck on one eager mid-config inference whose action-expert
# megakernel runs without CTA pairs (a plain cooperative launch the sanitizer can replay).
# Logs: gpurun_out/sanitize_*.log (summaries copied under profiles/).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --print-limit 20"
export PI0B_AE_PAIR=0 PI0B_AE_PAIR_FFN=0 PI0B_AE_SYM_QKV=0
for tool in memcheck racecheck synccheck; do
  timeout ${T_SAN:-900} $CS --tool $tool python scripts/sanitize_run.py 2 0 > gpurun_out/sanitize_engine_$tool.log 2>&1
  echo "engine $tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|max \|engine' gpurun_out/sanitize_engine_$tool.log | tr '\n' ' ')"
done
unset PI0B_AE_PAIR PI0B_AE_PAIR_FFN PI0B_AE_SYM_QKV
timeout ${T_SAN:-900} $CS --tool memcheck python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider > gpurun_out/sanitize_kernels_memcheck.log 2>&1
echo "kernel tests memcheck rc=$?: $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_kernels_memcheck.log | tail -3 | tr '\n' ' ')"
