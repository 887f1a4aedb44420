#!/bin/bash
# Sweep prefill GEMM tile width / split-K per node family (node_times per config).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for cfg in "128 0" "64 1" "64 2" "128 1" "128 2" "128 4" "256 1" "256 2" "256 4"; do
  set -- $cfg
  env=""
  for n in ${NODES:-VE_QKV VE_PROJ VE_FC1 VE_FC2}; do env="$env PI0B_BN_$n=$1 PI0B_SPLIT_$n=$2"; done
  echo "== bn=$1 split=$2"
  env $env timeout 120 python scripts/node_times.py 2 2>&1 | grep -E "^(ve|llm)\.|replay"
done
