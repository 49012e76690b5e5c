# usage: ab.sh name1=path1 name2=path2 ... (path "" = default lib)
for kv in "$@"; do
  n=${kv%%=*}; p=${kv#*=}
  for rep in 1 2; do
    SPCT_LIB_PATH=$p timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$n.log 2>&1
    tail -1 gpurun_out/ab_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['e2e']['value'])"
  done
done
