#!/bin/bash
# A/B of two builds of the library on one box: tools/ab.sh a.so b.so [rounds]
mkdir -p gpurun_out
for r in $(seq ${3:-2}); do
  for lib in "$1" "$2"; do
    SPCT_LIB_PATH=$lib python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; b=d.get('build_only') or {}; c=d.get('c5_batch') or {}
print('$lib', 'step', d['ms_per_step'], 'kernel', r['kernel_ms'], 'build', b.get('kernel_ms'), 'c5', c.get('ms_per_frame'))"
  done
done
