"""Summarise an ncu report's source page by CUDA source line.

python scripts/ncu_lines.py report.ncu-rep [top | first-last]
Prints the lines with the most warp-stall samples and executed instructions,
plus the dominant stall reasons per line.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    rng = None
    if len(sys.argv) > 2 and "-" in sys.argv[2]:  # a line range "a-b": print it in line order
        rng = tuple(int(x) for x in sys.argv[2].split("-"))
        top = 10 ** 9
    else:
        top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    for i, r in enumerate(rows):
        if r and r[0] == "Line No":
            hdr, start = r, i + 1
            break
    if hdr is None:
        print(out[:2000])
        return
    idx = {h: k for k, h in enumerate(hdr) if h not in idx} if False else {}
    for k, h in enumerate(hdr):
        idx.setdefault(h, k)
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {}
    total_s = 0
    for r in rows[start:]:
        if len(r) < len(hdr) or not r[0].strip().isdigit():
            continue
        line = int(r[0])
        src = r[1]
        try:
            s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
            ins = int(r[idx["Instructions Executed"]] or 0)
        except ValueError:
            continue
        a = agg.setdefault(line, {"src": src.strip(), "samples": 0, "inst": 0, "stalls": {}})
        a["samples"] += s
        a["inst"] += ins
        total_s += s
        for c in stall_cols:
            try:
                v = int(r[idx[c]] or 0)
            except ValueError:
                v = 0
            if v:
                a["stalls"][c[6:]] = a["stalls"].get(c[6:], 0) + v
    print(f"total samples {total_s}")
    items = sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]
    if rng:
        items = sorted((kv for kv in agg.items() if rng[0] <= kv[0] <= rng[1] and kv[1]["inst"]),
                       key=lambda kv: kv[0])
    for line, a in items:
        st = sorted(a["stalls"].items(), key=lambda kv: -kv[1])[:3]
        sts = " ".join(f"{k}={v}" for k, v in st)
        print(f"{line:5d} {100.0 * a['samples'] / max(total_s, 1):5.1f}% inst={a['inst']:>11d} "
              f"{sts:50s} | {a['src'][:70]}")


if __name__ == "__main__":
    main()
