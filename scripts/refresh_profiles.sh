#!/bin/bash
# GPU side of the round's profile refresh: bench lines of the three BASELINE configs, per-node
# times + megakernel trace (f4 calibration), streaming measurements (8(d)(iii), f2).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/refresh
for cfg in "1 0" "2 0" "3 32"; do
  set -- $cfg
  timeout 600 python bench.py --steps 200 --warmup 20 --views $1 --prompt $2 --no-cpu > gpurun_out/refresh/bench_${1}v${2}p.json 2>/dev/null
done
timeout 300 python scripts/node_times.py 2 > gpurun_out/refresh/node_times.txt 2>&1
cp gpurun_out/node_times.json gpurun_out/refresh/
timeout 300 python scripts/ae_trace.py 2 > gpurun_out/refresh/ae_trace.txt 2>&1
timeout 600 python scripts/stream_bench.py 2 > gpurun_out/refresh/stream_2v.json 2> gpurun_out/refresh/stream_2v.err
timeout 600 python scripts/stream_runtime.py 3 > gpurun_out/refresh/stream_runtime_2v.json 2> gpurun_out/refresh/stream_runtime.err
ls -la gpurun_out/refresh
