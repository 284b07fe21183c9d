import time, numpy as np
import paper_2302_11825_b200 as B
from paper_2302_11825_b200 import configs
c = configs.config2()
scene = B.Scene(c.vertices, c.segments, c.labels)
region = B.SolveRegion(scene, offset=c.region_offset, epsilon=c.epsilon)
for ms in [10000, 1000, 100]:
    cfg = c.cache; cfg.walk.maxSteps = ms
    st = {}
    t0 = time.time(); cache = B.generate_boundary_cache(scene, c.problem, region, cfg, 1, 0, stats=st); B.synchronize(); t1 = time.time()
    print("maxSteps", ms, st, "wall", round(t1 - t0, 3), flush=True)
cfg.walk.maxSteps = 10000
pb = c.problem
for x in [[0.0, -0.9995], [0.0, 0.0], [0.5, -0.5], [0.99, 0.99], [-0.9, -0.9995]]:
    wc = B.walk_config(epsilon=1e-3, nWalks=100000, seed=3)
    t0 = time.time(); e = B.wost_solve(scene, pb, [x], wc); t1 = time.time()
    print(x, e["mean"], e["se"], e["truncated"], "wall", round(t1 - t0, 3), flush=True)
