"""Where the end-to-end (host buffers) time of one C2 round goes."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = getattr(configs, f"config{cid}")()
scene = B.Scene(c.vertices, c.segments, c.labels)
region = B.SolveRegion(scene, offset=c.region_offset, epsilon=c.epsilon)
points = np.ascontiguousarray(c.points)
pinned = torch.from_numpy(points).pin_memory().numpy()
for label, src in (("pageable", points), ("pinned", pinned)):
    for k in range(4):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        pts = B.EvaluationPoints(src, 2)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        B.mark_evaluation_points(scene, region, c.cache, pts)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        B.update_solution(scene, c.problem, region, c.cache, pts, c.seed, 500 + k, gradients=True)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        u, g = pts.read_solution(gradient=True)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        d = np.diff(t) * 1e3
        if k:
            print(label, "create %.2f mark %.2f update %.2f read %.2f total %.2f ms" % (*d, sum(d)), flush=True)
