#!/bin/bash
# Per-node times (scripts/node_times.py) under several env configurations:
#   scripts/env_sweep.sh "NAME1:VAR=V VAR=V" "NAME2:..."
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for spec in "$@"; do
  name=${spec%%:*}; vars=${spec#*:}
  echo "== $name ($vars)"
  env $vars timeout 200 python scripts/node_times.py ${VIEWS:-2} 2>&1 | grep -E "^(ve|llm)\.|replay" | head -${TOPN:-14}
done
