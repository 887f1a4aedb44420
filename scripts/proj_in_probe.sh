#!/bin/bash
# llm.proj_in / ve.embed tile configurations (one-off GEMMs with fp32 + bf16 outputs): node time and replay.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in "" "PI0B_BN_LLM_PROJ_IN=128" "PI0B_BN_LLM_PROJ_IN=128 PI0B_SPLIT_LLM_PROJ_IN=1" "PI0B_BN_LLM_PROJ_IN=64" "PI0B_BN_VE_EMBED=64" "PI0B_BN_VE_EMBED=64 PI0B_SPLIT_VE_EMBED=1" "PI0B_SPLIT_VE_EMBED=1"; do
  echo "[$v] $(env $v timeout 300 python scripts/node_times.py 2 2>/dev/null | grep -E 'proj_in|ve.embed|graph replay' | tr -s ' ' | tr '\n' ';')"
done
