import time, numpy as np, torch
import paper_2302_11825_b200 as B
from paper_2302_11825_b200 import configs
c = configs.config2()
sc = B.Scene(c.vertices, c.segments, c.labels)
rg = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
pts0 = B.EvaluationPoints(c.points); B.mark_evaluation_points(sc, rg, c.cache, pts0)
B.update_solution(sc, c.problem, rg, c.cache, pts0, c.seed, 0, gradients=True)
for rep in range(3):
    t = [time.perf_counter()]
    pts = B.EvaluationPoints(c.points); torch.cuda.synchronize(); t.append(time.perf_counter())
    B.mark_evaluation_points(sc, rg, c.cache, pts); torch.cuda.synchronize(); t.append(time.perf_counter())
    B.update_solution(sc, c.problem, rg, c.cache, pts, c.seed, 1 + rep, gradients=True); torch.cuda.synchronize(); t.append(time.perf_counter())
    st = pts.download(); t.append(time.perf_counter())
    u = pts.solution(st); t.append(time.perf_counter())
    print("create %.1f mark %.1f update %.1f download %.1f solution %.1f ms" % tuple(1e3 * np.diff(t)))
for rep in range(3):
    t0 = time.perf_counter(); B.update_solution(sc, c.problem, rg, c.cache, pts0, c.seed, 10 + rep, gradients=True); torch.cuda.synchronize(); print("update on existing points %.1f ms" % (1e3 * (time.perf_counter() - t0)))
