#!/bin/bash
# p50 replay / e2e / action-expert time across view counts and prompt lengths (any prompt length
# runs on the default engine: the prefix is padded to 32-row multiples).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in 1 2 3; do for pr in 0 17 32 64 200; do
  echo "$v $pr $(timeout 300 python bench.py --views $v --prompt $pr --steps ${STEPS:-60} --warmup 5 --no-cpu 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['ms_per_launch'], d['step_roofline']['frac'], (d.get('parity') or {}).get('max_abs'))")"
done; done
