# usage: bash tools/spills.sh <file.cu> : registers / spills per kernel of one translation unit
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v -diag-suppress 177 $FL_EXTRA -c $1 -o /tmp/spills_$$.o 2>&1 | python3 -c "
import sys,re
name=None
for line in sys.stdin:
    m=re.search(r\"Compiling entry function '(\w+)'\",line)
    if m: name=m.group(1)
    m=re.search(r'(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads',line)
    if m and name: print(f'{m.group(2):>5} st {m.group(3):>5} ld  {name}')
"
