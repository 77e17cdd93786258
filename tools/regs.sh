#!/bin/bash
# Summarise ptxas register/spill usage per kernel instantiation (build/*.ptxas.txt).
python3 - "$@" <<'PY'
import re,sys
for fn in sys.argv[1:]:
    cur=None; sp=None
    for line in open(fn):
        m=re.search(r"Compiling entry function '(\S+)'", line)
        if m: cur=m.group(1); continue
        m=re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m: sp=(m.group(1), m.group(2)); continue
        m=re.search(r"Used (\d+) registers", line)
        if m and cur:
            k=re.search(r"op([23])d_kernelILi(\d)ELi(\d)ELi\d+ELb(\d)", cur)
            tag = f"{k.group(1)}D mode{k.group(2)} epi{k.group(3)} iso{k.group(4)}" if k else cur[:50]
            print(f"{tag:40s} regs={m.group(1):>4s} spill={sp}")
            cur=None
PY
