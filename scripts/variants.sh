#!/bin/bash
# A/B experiments: build variant libraries (here, on CPU) and time each on the GPU box.
#   build:  scripts/variants.sh build NAME "-DX=1 -DY=2" [NAME2 "..."]
#   run:    scripts/variants.sh run NAME... (on the box: AE trace summary + bench line per variant)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mode=$1; shift
if [ "$mode" = build ]; then
  while [ $# -gt 0 ]; do
    python paper_2510_26742_b200/build.py "variants/lib_$1.so" $2 || exit 1; shift 2
  done
else
  mkdir -p gpurun_out
  for v in "$@"; do
    lib=""; [ "$v" != base ] && lib="$PWD/variants/lib_$v.so"
    echo "=== $v"
    PI0B_LIB=$lib timeout 300 python scripts/ae_trace.py ${VIEWS:-2} > gpurun_out/trace_$v.txt 2>&1; head -${TL:-8} gpurun_out/trace_$v.txt
    if [ -n "$BENCH" ]; then
      PI0B_LIB=$lib timeout 300 python bench.py --steps 50 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], 'e2e', d['e2e']['value'], 'ae', d['roofline']['ms_per_launch'])"
    fi
  done
fi
