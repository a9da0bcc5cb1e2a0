#!/bin/bash
# print kernel: registers spill-bytes
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 -Xptxas -v -c -o /tmp/x.o paper_1912_02949_b200/csrc/sketchycgal.cu 2>&1 | python3 -c "
import sys,re
name=None
for line in sys.stdin:
    m=re.search(r\"entry function '_ZN3scg\d+([a-z_]+)\",line)
    if m: name=m.group(1); spill=None; continue
    m=re.search(r'(\d+) bytes spill stores',line)
    if m: spill=m.group(1)
    m=re.search(r'Used (\d+) registers',line)
    if m and name: print(f'{name:16s} regs={m.group(1):4s} spill={spill}'); name=None
    if 'error' in line: print(line.strip())
"
