"""Per-phase instruction / stall-sample shares of an ncu report.

python scripts/ncu_phases.py report.ncu-rep file.cu name:line [name:line ...]
Each name:line starts a phase that runs until the next one (lines of file.cu);
lines of other files (inlined helpers) are reported per file.
"""
import csv
import io
import subprocess
import sys


def main():
    rep, fname = sys.argv[1], sys.argv[2]
    marks = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[3:]]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr, data = None, None, {}
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and r and r[0].strip().isdigit() and len(r) >= len(hdr):
            try:
                v = int(r[hdr.index("Instructions Executed")] or 0)
                s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            except ValueError:
                continue
            a = data.setdefault((cur, int(r[0])), [0, 0])
            a[0] += v
            a[1] += s
    tot = sum(v[0] for v in data.values()) or 1
    tots = sum(v[1] for v in data.values()) or 1
    bounds = marks + [("end", 10 ** 9)]
    acc = {}
    for (f, l), (v, s) in data.items():
        if f != fname:
            key = "[" + f + "]"
        else:
            key = "pre"
            for (n, a), (_, b) in zip(bounds, bounds[1:]):
                if a <= l < b:
                    key = n
        x = acc.setdefault(key, [0, 0])
        x[0] += v
        x[1] += s
    print(f"total warp instructions {tot:.4g}")
    for k, (v, s) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
        print(f"{k:28s} inst {100 * v / tot:5.1f}%  samples {100 * s / tots:5.1f}%")


if __name__ == "__main__":
    main()
