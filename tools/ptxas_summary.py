"""Summarise nvcc -Xptxas -v output: kernel, registers, spill stores/loads (filter by a substring)."""
import re
import sys

cur = None
rows = []
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '([^']*)'", line)
    if m:
        cur = [m.group(1), None, None, None]
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur[2], cur[3] = int(m.group(1)), int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur[1] = int(m.group(1))
for name, regs, ss, sl in rows:
    if pat in name:
        print("%-70s regs %4s spill %5s/%5s" % (name[:70], regs, ss, sl))
