"""Registers / spills per kernel from an nvcc -Xptxas -v log.
python scripts/ptxas_table.py build/ball12.ptxas.log [filter]"""
import re
import sys

cur = None
rows = {}
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        rows.setdefault(cur, {})["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for k in sorted(rows):
    if flt in k:
        short = re.sub(r"^_ZN3vxb\d*\w*?(\w+_kernel)I(.*?)EEEv.*$", r"\1<\2>", k)
        print(f"{short:40s} regs {rows[k].get('regs')} spill {rows[k].get('spill')}")
