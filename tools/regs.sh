#!/bin/bash
# Register / spill summary of the fused sweep variants of one translation unit.
#   tools/regs.sh paper_1711_01656_b200/csrc/fused_kw64_s1.cu
f=${1:-paper_1711_01656_b200/csrc/fused_kw64_s1.cu}
/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Iinclude -Ipaper_1711_01656_b200/csrc -c "$f" -o /tmp/regs.o -Xptxas -v 2>&1 |
python3 -c "
import re,sys
cur=None
for line in sys.stdin:
    m=re.search(r\"Compiling entry function '(\S+)'\",line)
    if m: cur=m.group(1); continue
    m=re.search(r'(\d+) bytes spill stores, (\d+) bytes spill loads',line)
    if m and cur: spill=m.group(0); continue
    m=re.search(r'Used (\d+) registers',line)
    if m and cur:
        t=re.search(r'sweep_match_kernelIL(b[01])EL(i\d)EL(i\d+)EL(b[01])EL(i\d)EL(i\d)E',cur)
        name=('STORE=%s MODE=%s KW=%s ALLB=%s SK=%s S=%s'%t.groups()) if t else cur[:60]
        print(name, 'regs', m.group(1), '|', spill); cur=None
" | sort
