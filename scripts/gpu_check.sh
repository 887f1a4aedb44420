#!/bin/bash
# One gpurun session: environment facts, kernel + engine parity tests, smoke.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nvidia-smi -L; nproc; lscpu | grep -E "Model name|^CPU\(s\)"; free -g | head -2; } > gpurun_out/env.txt 2>&1
timeout ${T_KERNELS:-300} python -m pytest tests/test_gpu_kernels.py -q --timeout=120 --timeout-method=thread ${KSEL:+-k "$KSEL"} > gpurun_out/kernels.log 2>&1
timeout ${T_ENGINE:-500} python -m pytest tests/test_gpu_engine.py -q -s --timeout=240 --timeout-method=thread ${ESEL:+-k "$ESEL"} > gpurun_out/engine.log 2>&1
tail -30 gpurun_out/kernels.log; tail -40 gpurun_out/engine.log
if [ -n "$BENCH" ]; then
  timeout 600 python bench.py --steps ${STEPS:-20} --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
fi
