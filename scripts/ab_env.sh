#!/bin/bash
# A/B of environment switches on one box: bench value / e2e / AE ms, alternating (ROUNDS times).
# usage: scripts/ab_env.sh "" "PI0B_X=0" "PI0B_X=0 PI0B_Y=1" ...   ("" = defaults)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in $(seq ${ROUNDS:-2}); do
  for v in "$@"; do
    echo "[$v] $(env $v timeout 300 python bench.py --steps ${STEPS:-100} --warmup 10 --no-cpu ${BENCH_ARGS} 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'e2e', d['e2e']['value'], 'ae', d['roofline']['ms_per_launch'])")"
  done
done
