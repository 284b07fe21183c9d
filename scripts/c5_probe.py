import time, numpy as np, torch
import paper_2302_11825_b200 as B
from paper_2302_11825_b200 import configs
c = configs.config5(scale=1/16, n_points=200000)
t0 = time.time()
tris, labels = configs.soup_shell(c)
comps = configs.soup_components(c)
keep = np.zeros(len(c.points), bool)
for m in comps: keep |= m.inside(c.points)
pts_x = c.points[keep][:200000]
sc = B.Scene.mesh3(c.vertices, tris, labels)
region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
print("setup", time.time() - t0, "shell tris", len(tris), "of", len(c.segments), "points", len(pts_x), "closed-mesh inside? ", flush=True)
pts = B.EvaluationPoints(pts_x, 3)
B.mark_evaluation_points(sc, region, c.cache, pts)
for r in range(2):
    torch.cuda.synchronize(); t = time.time()
    st = B.update_solution(sc, c.problem, region, c.cache, pts, c.seed, r)
    torch.cuda.synchronize(); print("round", r, st, time.time() - t, flush=True)
s = pts.download(); u = pts.solution(s)
print("u range", np.nanmin(u), np.nanmax(u), "pct", np.percentile(u, [1, 50, 99]), "fallback", s["fallback"].sum())
# self-consistency: pointwise walks at a few interior points vs BVC
