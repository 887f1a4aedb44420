#!/bin/bash
# Round-end style GPU pass: the whole -m gpu suite (measured parity -> gpurun_out/parity/*.json),
# then the bench.  TSAN=1 adds the compute-sanitizer pass.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/parity
[ -n "$TSAN" ] && bash scripts/sanitize.sh
PI0B_PARITY_OUT=gpurun_out/parity timeout ${T_TESTS:-1500} python -m pytest tests -m gpu -q -s -rA --timeout=600 ${TSEL:+-k "$TSEL"} > gpurun_out/tests.log 2>&1
grep -E "^(PASSED|FAILED|ERROR)|passed|failed" gpurun_out/tests.log | tail -100
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py --steps ${STEPS:-200} --warmup 20 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
fi
