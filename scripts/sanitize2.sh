#!/bin/bash
# compute-sanitizer over the kernels changed in round 2: prefill attention (128-key tiles, key
# splits through the L2 workspace, padded key segments), the staged residual GEMM epilogue, the
# view-sharded VE push / wait kernels (two shard engines on one device) and unaligned prompts.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CS="compute-sanitizer --target-processes all --print-limit 20"
for tool in memcheck racecheck synccheck; do
  timeout ${T_SAN:-900} $CS --tool $tool python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "attention or residual" > gpurun_out/sanitize2_kernels_$tool.log 2>&1
  echo "kernels $tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitize2_kernels_$tool.log | tail -2 | tr '\n' ' ')"
done
# (the one-device view-shard test cannot run under the sanitizer: it serialises kernels, so a shard
# engine's wait kernel spins on a peer stream that never runs and traps after 10 s)
export PI0B_AE_PAIR=0 PI0B_AE_PAIR_FFN=0 PI0B_AE_SYM_QKV=0
for tool in memcheck racecheck; do
  timeout ${T_SAN:-900} $CS --tool $tool python scripts/sanitize_run.py 1 17 > gpurun_out/sanitize2_prompt17_$tool.log 2>&1
  echo "engine 1v+17p $tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|max \|engine' gpurun_out/sanitize2_prompt17_$tool.log | tr '\n' ' ')"
done
