#!/bin/bash
# A/B on one box: bench value / e2e / AE ms for each library, alternating (ROUNDS times).
# usage: scripts/ab_bench.sh variants/lib_a.so [variants/lib_b.so ...]   ("base" = in-tree lib)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in $(seq ${ROUNDS:-2}); do
  for v in "$@"; do
    lib=""; [ "$v" != base ] && lib="$PWD/$v"
    PI0B_LIB=$lib timeout 300 python bench.py --steps ${STEPS:-100} --warmup 10 --no-cpu ${BENCH_ARGS} 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'value', d['value'], 'e2e', d['e2e']['value'], 'ae', d['roofline']['ms_per_launch'])"
  done
done
