#!/bin/bash
# llm.attn key splits across prefix lengths (bench value per setting).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for cfg in "2 17" "3 0" "3 32" "1 17" "2 64"; do set -- $cfg
  for s in 1 2 4; do
    echo "$1v$2p S=$s $(PI0B_ATTN_SPLITS_LLM_ATTN=$s timeout 300 python bench.py --views $1 --prompt $2 --steps 40 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])")"
  done
done
