"""Instruction mix of every backward-branch loop of one kernel's SASS.
python scripts/sass_loops.py file.(o|so|cubin) kernel_substring"""
import re
import subprocess
import sys
from collections import Counter

obj, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ins = []
    for l in f.split("\n"):
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    print(name, len(ins), "instructions")
    for a, t in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?(0x[0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            tgt = int(m.group(1), 16)
            body = [x for x in ins if tgt <= x[0] <= a]
            c = Counter(re.sub(r"^@!?U?P\w+\s+", "", x[1]).split()[0].split(".")[0] for x in body)
            print(f"  loop {tgt:#x}-{a:#x}: {len(body)}", dict(c.most_common(14)))
