#!/bin/bash
# One gpurun session: tests, bench, launch list (+ optional ncu --set full of one kernel).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nvidia-smi -L; nproc; lscpu | grep -E "Model name|^CPU\(s\)"; free -g | head -2; ldd --version | head -1; } > gpurun_out/env.txt 2>&1
if [ -z "$NOTEST" ]; then
  timeout ${T_TESTS:-900} python -m pytest tests -m gpu -x -q -s -rA --timeout=300 ${TSEL:+-k "$TSEL"} > gpurun_out/tests.log 2>&1
  tail -15 gpurun_out/tests.log
fi
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py --steps ${STEPS:-50} --warmup 10 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
fi
if [ -n "$NODES" ]; then
  timeout 300 python scripts/node_times.py ${VIEWS:-2} > gpurun_out/node_times.txt 2>&1; cat gpurun_out/node_times.txt
fi
if [ -n "$LAUNCHES" ]; then
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches.csv python scripts/ncu_launches.py ${VIEWS:-2} > gpurun_out/launches.log 2>&1
  tail -2 gpurun_out/launches.log
fi
if [ -n "$FULL" ]; then   # FULL="<kernel regex>" ; SKIP = launches to skip
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"$FULL" \
     -s ${SKIP:-0} -c ${COUNT:-1} -f -o gpurun_out/prof python scripts/ncu_launches.py ${VIEWS:-2} > gpurun_out/full.log 2>&1
  tail -3 gpurun_out/full.log
fi
