import time, numpy as np
import paper_2302_11825_b200 as B
from paper_2302_11825_b200 import configs
c = configs.config2()
scene = B.Scene(c.vertices, c.segments, c.labels)
region = B.SolveRegion(scene, offset=c.region_offset, epsilon=c.epsilon)
pts = B.EvaluationPoints(c.points)
B.mark_evaluation_points(scene, region, c.cache, pts)
for r in range(3):
    t0 = time.time(); st = B.update_solution(scene, c.problem, region, c.cache, pts, c.seed, r, gradients=True); t1 = time.time()
    print("C2 round", r, st, "wall", round(t1 - t0, 4), flush=True)
s = pts.download(); u = pts.solution(s); g = pts.gradient(s)
fb = s["fallback"]
print("fallback", fb.sum(), "u rmse", np.sqrt(np.mean((u - c.points[:, 0]) ** 2)), "u rmse nonfb", np.sqrt(np.mean((u[~fb] - c.points[~fb, 0]) ** 2)))
gi = ~fb & ~s["gradientUnreliable"]
print("grad rmse", np.sqrt(np.mean((g[gi] - [1, 0]) ** 2, axis=0)), "mean grad", g[gi].mean(0))
print("launches", B.launch_count())
