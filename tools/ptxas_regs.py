"""Print (kernel, registers, spills) from a ptxas -v log: python tools/ptxas_regs.py LOG [substr]."""
import re
import sys

cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m:
        spill = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and (len(sys.argv) < 3 or sys.argv[2] in cur):
        print(m.group(1), "regs", "spill=" + spill, cur)
        cur = None
