"""Per-source-line instruction / stall breakdown of one kernel in an ncu report.
python scripts/ncu_src.py report.ncu-rep kernel_regex [min_pct] [units]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
minp = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
units = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
for i, r in enumerate(rows):
    if r and r[0] == "Line No":
        hdr, start = r, i + 1
        break
ix = {}
for k, h in enumerate(hdr):
    ix.setdefault(h, k)
agg = []
tot = tots = 0
for r in rows[start:]:
    if len(r) < len(hdr) or not r[0].strip().isdigit():
        continue
    try:
        ins = int(r[ix["Instructions Executed"]] or 0)
        smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    if ins or smp:
        agg.append((int(r[0]), ins, smp, r[1].strip()[:95]))
        tot += ins
        tots += smp
print(f"total inst {tot:.4g}  samples {tots}")
for ln, ins, smp, src in sorted(agg):
    if ins > minp / 100 * tot or smp > minp / 100 * tots:
        per = f" {ins / units:7.1f}/u" if units else ""
        print(f"{ln:5d} {100 * ins / tot:5.1f}% {100 * smp / max(tots, 1):5.1f}%s{per} | {src}")
