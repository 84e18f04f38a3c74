#!/bin/bash
# Rebuild the library and summarise ptxas register/spill use of the cell-map kernels.
cd "$(dirname "$0")/.." && touch paper_1802_05246_b200/csrc/cellmap.cuh && make -j12 PTXAS="-Xptxas -v" 2>&1 | python3 -c "
import sys,re
cur=None
for line in sys.stdin:
    if 'error' in line: print(line.rstrip())
    m=re.search(r\"Compiling entry function '(\S+)'\",line)
    if m: cur=m.group(1); continue
    if cur and 'cellmap' in cur:
        m2=re.search(r'(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads',line)
        if m2: st=m2.groups()
        m3=re.search(r'Used (\d+) registers',line)
        if m3:
            k=re.search(r'ILi(\d)ELi(\d)',cur).groups(); print('m=%s sch=%s regs=%s stack/spill=%s'%(k[0],k[1],m3.group(1),st)); cur=None
" | sort
