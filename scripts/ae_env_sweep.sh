#!/bin/bash
# AE megakernel span (scripts/ae_trace.py) under several env configurations:
#   scripts/ae_env_sweep.sh "NAME1:VAR=V VAR=V" "NAME2:..."
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for spec in "$@"; do
  name=${spec%%:*}; vars=${spec#*:}
  [ "$vars" = "$spec" ] && vars=""
  printf "%-14s %-50s " "$name" "$vars"
  env $vars timeout 200 python scripts/ae_trace.py ${VIEWS:-2} 2>&1 | grep -m1 span | sed 's/.*span/span/'
done
