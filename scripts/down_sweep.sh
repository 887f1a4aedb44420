cd "${GRAFT_REPO_ROOT:-/root/repo}"
for cfg in "1 0" "3 0" "3 32" "2 17"; do set -- $cfg
  for v in "" "PI0B_BN_LLM_DOWN=256 PI0B_SPLIT_LLM_DOWN=2" "PI0B_BN_LLM_DOWN=256 PI0B_SPLIT_LLM_DOWN=3" "PI0B_BN_LLM_DOWN=256 PI0B_SPLIT_LLM_DOWN=4" "PI0B_SPLIT_LLM_DOWN=3" "PI0B_SPLIT_LLM_DOWN=4"; do
    echo "$1v$2p [$v] $(env $v timeout 300 python bench.py --views $1 --prompt $2 --steps 40 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'])")"
  done
done
