"""Does spatial coherence within a warp speed up BVH queries enough to pay for sorting
walkers? Closest-Dirichlet-point queries on C4's mesh for 4M walker-like points (cache
sample positions moved inward by exponential depths), in random order and in Morton
order; time the query kernel with ncu (closest3_kernel).
    ncu --metrics gpu__time_duration.sum -k regex:closest3 python scripts/coherence_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402

c = configs.config4()
sc = B.Scene.mesh3(c.vertices, c.segments, c.labels)
region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
cache = B.generate_boundary_cache(sc, c.problem, region, c.cache, c.seed, 0).download()
rng = np.random.default_rng(0)
n = 1 << 22
idx = rng.integers(0, len(cache["z"]), n)
depth = rng.exponential(0.03, n)
x = cache["z"][idx] - depth[:, None] * cache["n"][idx]


def morton(p):
    lo, hi = p.min(0), p.max(0)
    q = ((p - lo) / (hi - lo) * 1023).astype(np.uint64)
    key = np.zeros(len(p), np.uint64)
    for b in range(10):
        for a in range(3):
            key |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
    return key


shuffled = x[rng.permutation(n)]
sorted_ = x[np.argsort(morton(x))]
for name, pts in (("random", shuffled), ("morton", sorted_), ("random", shuffled), ("morton", sorted_)):
    _, d, _, _ = sc.closest_point(pts, abi.FILTER_DIRICHLET)
    print(name, float(np.mean(d)), flush=True)
