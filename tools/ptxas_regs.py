"""Registers / spills per kernel from an `nvcc -Xptxas -v` log: python tools/ptxas_regs.py log [filter]"""
import re
import subprocess
import sys

txt = open(sys.argv[1]).read()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for m in re.finditer(r"Compiling entry function '(\S+)' for.*?\n.*?\n\s+(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads\n.*?Used (\d+) registers", txt):
    name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
    name = re.sub(r"\(spaimg::Layout.*", "", name)
    if flt in name:
        print(f"{int(m.group(5)):4d} regs  stack {m.group(2):>4}  spill st/ld {m.group(3)}/{m.group(4)}  {name}")
