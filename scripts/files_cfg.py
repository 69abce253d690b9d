"""Time vx_tessellate_to_files on a baseline config (row f2 streaming).
python scripts/files_cfg.py K [dir] [reps] [--dist]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2201_13234_b200 as vx  # noqa: E402

k = int(sys.argv[1])
d = sys.argv[2] if len(sys.argv) > 2 else "/tmp"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
with_dist = "--dist" in sys.argv
p = oracle.baseline_config(k)
box = vx.Domain(p.lengths, vx.Boundary.Periodic if p.periodic else vx.Boundary.NonPeriodic)
grid = vx.VoxelGrid(p.counts, box)
sites = vx.SiteSet(vx.Kind(p.kind), p.dim, p.positions, p.times, p.growth)
lab = os.path.join(d, f"cfg{k}.lab")
dist = os.path.join(d, f"cfg{k}.dist") if with_dist else None
for r in range(reps):
    t0 = time.perf_counter()
    vx.tessellate_to_files(sites, grid, lab, dist, seed=1000 + k)
    dt = time.perf_counter() - t0
    nbytes = os.path.getsize(lab) + (os.path.getsize(dist) if dist else 0)
    print(f"cfg{k} to_files {dt * 1e3:.1f} ms  {nbytes / dt / 1e9:.2f} GB/s written  "
          f"{p.n_voxels / dt / 1e9:.2f} Gvox/s", flush=True)
im, meta = vx.read_label_image(lab)
fp = oracle.fingerprint(im.labels.view("int32"))
print(f"fingerprint {fp} {'OK' if fp == oracle.SURVEY_FINGERPRINTS[k] else 'FAIL'}")
os.remove(lab)
os.remove(lab + ".json")
if dist:
    os.remove(dist)
    os.remove(dist + ".json")
