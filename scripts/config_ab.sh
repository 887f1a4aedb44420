#!/bin/bash
# A/B of libraries across the BASELINE configs and a few prompt lengths (bench value, p50 ms).
# usage: LIBS="variants/lib_x.so ..." scripts/config_ab.sh   ("base" = the in-tree library)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for cfg in "1 0" "2 0" "3 32" "2 17" "3 0" "1 17"; do set -- $cfg
  for v in base ${LIBS}; do
    L=""; [ "$v" != base ] && L="$PWD/$v"
    echo "$1v$2p $v $(PI0B_LIB=$L timeout 300 python bench.py --views $1 --prompt $2 --steps ${STEPS:-40} --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], (d.get('parity') or {}).get('max_abs'))")"
  done
done
