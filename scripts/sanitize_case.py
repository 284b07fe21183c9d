"""Small cases of every round path for compute-sanitizer (memcheck): the smoke round,
a clamp-corrected round, a 3D mixed round on a small displaced sphere, and a 1-rank
sharded round through a host-staged communicator.
    compute-sanitizer --tool memcheck python scripts/sanitize_case.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as G  # noqa: E402
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402
from tests import helpers as H  # noqa: E402

G.smoke()
geom, pb = H.disk_linear()
sc = B.Scene(*geom)
region = B.SolveRegion(sc, epsilon=1e-3 * sc.diagonal)
cfg = B.cache_config(clampMode=abi.CLAMP_CORRECT, clamp=0.05, nBoundary=256, nWalksNeumann=16, nWalksDirichlet=64,
                     correctionWalks=4)
p = B.EvaluationPoints(np.array([[0.9, 0.1], [0.5, -0.3]]))
B.mark_evaluation_points(sc, region, cfg, p)
B.update_solution(sc, pb, region, cfg, p, 3, 0, gradients=True)
c = configs.config5(scale=1 / 256, n_points=2000)
tris, labels = configs.soup_shell(c)
s3 = B.Scene.mesh3(c.vertices, tris, labels)
r3 = B.SolveRegion(s3, offset=c.region_offset, epsilon=c.epsilon)
cfg3 = c.cache
cfg3.nBoundary = 2048
x3 = c.points[:2000]
p3 = B.EvaluationPoints(x3, 3)
B.mark_evaluation_points(s3, r3, cfg3, p3)
B.update_solution(s3, c.problem, r3, cfg3, p3, 5, 0)
comm = B.Communicator.from_allgather(1, 0, lambda a, b, n: None)
geom2, pb2 = H.square_mixed()
sc2 = B.Scene(*geom2)
region2 = B.SolveRegion(sc2, offset=0.02, epsilon=1e-3 * sc2.diagonal)
cfg2 = B.cache_config(nBoundary=1001, nWalksNeumann=16, nWalksDirichlet=32, offset=0.02)
p2 = B.EvaluationPoints(np.random.default_rng(1).uniform(0.01, 0.99, (500, 2)))
B.mark_evaluation_points(sc2, region2, cfg2, p2)
B.update_solution_sharded(comm, sc2, pb2, region2, cfg2, p2, 9, 0, gradients=True)
print("sanitize case ok")
