import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, paper_2201_13234_b200 as vx
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from dev_check import random_instance, to_vx
rng = np.random.default_rng(12345)
p = random_instance(rng, 0)
print(p.dim, p.kind, p.periodic, p.counts, p.n_sites, flush=True)
sites, grid = to_vx(p)
eng = sys.argv[1]
r = vx.tessellate_fast(sites, grid) if eng == "fast" else vx.tessellate_brute(sites, grid)
lab, dist = oracle.brute(p)
print(eng, np.array_equal(r.labels.labels, lab), r.stats)
