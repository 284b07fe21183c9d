"""Where the end-to-end (host buffers) time of one round goes: the handle sequence's
pieces (create points from pinned memory, mark, updateSolution, read u) against one
bvc_update_solution_host call (the bench's e2e, pieces overlapped).
    python scripts/e2e_breakdown.py [config]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c, scene, region = bench.build_problem(cid, B, configs, abi)
grad = bool(c.gradients)
pinned = torch.from_numpy(np.ascontiguousarray(c.points)).pin_memory().numpy()
u_out = torch.empty(len(pinned), dtype=torch.float64).pin_memory().numpy()
g_out = torch.empty((len(pinned), c.dim), dtype=torch.float64).pin_memory().numpy() if grad else None
for k in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    pts = B.EvaluationPoints(pinned, c.dim)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    B.mark_evaluation_points(scene, region, c.cache, pts)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    st = B.update_solution(scene, c.problem, region, c.cache, pts, c.seed, 500 + k, gradients=grad)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    pts.read_solution(gradient=grad)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    del pts
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    B.update_solution_host(scene, c.problem, region, c.cache, pinned, c.seed, 600 + k, gradients=grad, out=(u_out, g_out))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if k:
        print("C%d pieces: create %.1f mark %.1f update %.1f (gen %.1f splat %.1f) read %.1f free %.1f = %.1f ms; "
              "host call %.1f ms" % (cid, *d[:3], st["generateSeconds"] * 1e3, st["splatSeconds"] * 1e3, *d[3:], sum(d),
                                     (t1 - t0) * 1e3), flush=True)
