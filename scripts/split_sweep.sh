#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for ms in 1 2 4 8 1000; do echo "== PI0B_MAX_SPLITS=$ms"; PI0B_MAX_SPLITS=$ms python scripts/node_times.py 2 2>&1 | grep -E "ae\.|ve.proj|llm.proj |llm.down|graph"; done
for ac in 8 16 32 128; do echo "== PI0B_ATTN_CTAS=$ac"; PI0B_ATTN_CTAS=$ac python scripts/node_times.py 2 2>&1 | grep -E "attn|graph"; done
