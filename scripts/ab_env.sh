cd "${GRAFT_REPO_ROOT:-/root/repo}"
for r in 1 2; do
for v in "lib_ab" "cur" "cur PI0B_AE_YDOUBLE=0" "cur PI0B_AE_PAIR_HEAD=0" "cur PI0B_AE_YDOUBLE=0 PI0B_AE_PAIR_HEAD=0"; do
  set -- $v; lib=$1; shift
  L=""; [ $lib = lib_ab ] && L=$PWD/variants/lib_ab.so
  echo "$v: $(env PI0B_LIB=$L "$@" timeout 300 python bench.py --steps 150 --warmup 10 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['ms_per_launch'])")"
done; done
