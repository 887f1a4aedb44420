#!/bin/bash
# Megakernel grid below the SM count (PI0B_AE_CTAS): single-inference latency and the streaming
# runtime (480 Hz and 1440 Hz 1-step ticks with a concurrent 30 Hz prefix).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for n in ${CTAS:-148 136 128 112}; do
  echo "== PI0B_AE_CTAS=$n"
  PI0B_AE_CTAS=$n timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  value', d['value'], 'ae', d['roofline']['ms_per_launch'])"
  PI0B_AE_CTAS=$n timeout 300 python scripts/stream_runtime.py 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
for r in d['runs']:
    print('  %6.0f Hz %-12s ticks/s %7.1f frames/s %5.2f quick %6.3f ms slow %6.2f ms prefix p50 %6.2f ms tick p50 %6.3f ms' % (
        r['ae_rate_target'], r['kv_policy'], r['ae_per_s'], r['vlm_per_s'], r['quick_mean_ms'], r['slow_mean_ms'], r['prefix_p50_ms'], r['tick_p50_ms']))"
done
