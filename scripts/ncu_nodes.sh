#!/bin/bash
# ncu --set full captures of the first launch of selected nodes (one GPU, one kernel each).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
NODES=${NODES:-"ae.qkv:gemm_tc ae.down:gemm_tc ve.qkv:gemm_tc llm.ffn:gemm_tc ae.attn:attn_kernel"}
for spec in $NODES; do
  node=${spec%%:*}; kern=${spec##*:}
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$kern -c 1 \
      -o gpurun_out/prof_${node} -f python scripts/ncu_node.py $node > gpurun_out/ncu_${node}.log 2>&1
  tail -2 gpurun_out/ncu_${node}.log
done
