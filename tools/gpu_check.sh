#!/bin/bash
# One GPU round trip: parity tests, smoke, a short bench; compact summary on stdout.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/pytest_gpu.log)"
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke: $(tail -1 gpurun_out/smoke.log)"
python bench.py --steps ${STEPS:-10} --warmup 3 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; b=d.get('build_only') or {}
print('bench:', d['value'], 'ms/step', d['ms_per_step'], 'kernel_ms', r['kernel_ms'], 'frac', r['frac'], 'e2e', d['e2e']['value'])
print('build_only:', b.get('value'), 'ms/step', b.get('ms_per_step'), 'kernel_ms', b.get('kernel_ms'), 'frac', b.get('frac'))
c=d.get('c5_batch') or {}; print('c5:', c.get('value'), 'ms/frame', c.get('ms_per_frame'))" 2>&1 | tail -3
