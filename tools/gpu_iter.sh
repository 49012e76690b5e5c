#!/bin/bash
# One GPU iteration: -m gpu tests (optional), launch lists of chosen workloads, a short bench.
#   TESTS=1 WORKLOADS="c3 c4 tmatch" BENCH_ARGS="--no-c5" bash tools/gpu_iter.sh
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc $? : $(tail -1 gpurun_out/pytest_gpu.log)"
  grep -E "^(FAILED|ERROR)|Error|assert" gpurun_out/pytest_gpu.log | head -20
fi
for m in ${WORKLOADS}; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$m.csv \
    python tools/workload_once.py $m 2 > gpurun_out/wo_$m.log 2>&1 || { echo "workload $m failed"; tail -5 gpurun_out/wo_$m.log; }
done
if [ -n "${BENCH_ARGS+x}" ]; then
  timeout 900 python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
  echo "bench rc $?"; tail -c 300 gpurun_out/bench.log | tail -2 | cut -c1-300
fi
