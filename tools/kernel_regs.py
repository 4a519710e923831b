#!/usr/bin/env python
"""Registers / stack (spill) bytes of the row-contiguous SpMMV kernels in the built
library (cuobjdump -res-usage), demangled: python tools/kernel_regs.py [filter]"""
import re
import subprocess
import sys

lib = "paper_1507_08101_b200/lib/libsellkit_b200.so"
out = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
flt = sys.argv[1] if len(sys.argv) > 1 else "spmv_tma_rows_kernel"
names = re.findall(r"Function ([^\s:]+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+)", out)
rows = []
for mangled, reg, stack, sh in names:
    dem = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
    if flt in dem:
        rows.append((dem.split("(")[0].replace("skb::spmv_detail::", ""), int(reg), int(stack), int(sh)))
for r in sorted(set(rows)):
    print(f"{r[0]:80s} REG {r[1]:3d} STACK {r[2]:4d} SHARED {r[3]}")
