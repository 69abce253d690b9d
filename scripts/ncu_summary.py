"""Write the dominant kernel's per-launch numbers from an `ncu --set full`
report into profiles/ncu_summary.json (read by bench.py for roofline.traffic).

python scripts/ncu_summary.py report.ncu-rep cfgK "kernel label"
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "duration_ns": "gpu__time_duration.sum",
    "registers": "launch__registers_per_thread",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issued_ipc": "sm__inst_issued.avg.per_cycle_active",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "warp_instructions": "smsp__inst_executed.sum",
}


def raw(rep):
    """Per-kernel metric dicts of every launch in the report."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?", one(hdr, units, vals))
            for vals in rows[2:] if len(vals) == len(hdr)]


def one(hdr, units, vals):
    res = {}
    for k, m in METRICS.items():
        if m in hdr:
            i = hdr.index(m)
            v = float(vals[i].replace(",", ""))
            u = units[i]
            byte_units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
            time_units = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}
            if k.startswith("dram") and u in byte_units:
                v *= byte_units[u]
            if k == "duration_ns" and u in time_units:
                v *= time_units[u]
            res[k] = v
    return res


def summarise(r):
    return {
        "dram_read_bytes": r.get("dram_read_bytes"),
        "dram_write_bytes": r.get("dram_write_bytes"),
        "duration_ms_under_ncu": r.get("duration_ns", 0.0) / 1e6,
        "registers": r.get("registers"),
        "achieved_occupancy_pct": r.get("achieved_occupancy_pct"),
        "issued_ipc": r.get("issued_ipc"),
        "fp64_pipe_pct": r.get("fp64_pipe_pct"),
        "warp_instructions": r.get("warp_instructions"),
    }


def main():
    rep, cfg, label = sys.argv[1], sys.argv[2], sys.argv[3]
    launches = raw(rep)
    total = lambda k: sum(r.get(k, 0.0) or 0.0 for _, r in launches)  # noqa: E731
    entry = {
        "kernel": label,
        "report": os.path.basename(rep),
        # one ball phase = every kernel launch captured in the report
        "ball_dram_bytes_per_launch": total("dram_read_bytes") + total("dram_write_bytes"),
        "dram_read_bytes": total("dram_read_bytes"),
        "dram_write_bytes": total("dram_write_bytes"),
        "duration_ms_under_ncu": total("duration_ns") / 1e6,
        "warp_instructions": total("warp_instructions"),
        "kernels": {name.split("<")[0].split("(")[0].split("::")[-1].split()[-1]: summarise(r) for name, r in launches},
    }
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    d = {}
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
    d["note"] = ("per-launch numbers of the dominant kernel from one `ncu --set full --clock-control none` "
                 "capture (cold caches, serialised; share of the step, not absolute time)")
    d[cfg] = entry
    with open(path, "w") as f:
        json.dump(d, f, indent=1)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
