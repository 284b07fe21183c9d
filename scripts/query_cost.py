"""Closest-Dirichlet-point query cost vs distance to the boundary (C2, C4, C5 scenes).

Times Scene.closest_point on same-size batches of interior points binned by their
distance to the boundary; the host transfers are identical per batch, so the
differences between bins are traversal cost."""
import sys, time
import numpy as np
import paper_2302_11825_b200 as B
from paper_2302_11825_b200 import abi, configs

def run(name, sc, pts, n=1 << 20, dim=3):
    _, d, _, _ = sc.closest_point(pts, abi.FILTER_DIRICHLET)
    dm = d.max()
    edges = [0, 0.002, 0.01, 0.03, 0.1, 0.2, 0.4, 0.7, 1.01]
    base = None
    for lo, hi in zip(edges[:-1], edges[1:]):
        sel = pts[(d >= lo * dm) & (d < hi * dm)]
        if len(sel) < 1000: continue
        x = sel[np.random.default_rng(0).integers(0, len(sel), n)]
        sc.closest_point(x[:1000], abi.FILTER_DIRICHLET)
        ts = []
        for _ in range(3):
            t = time.perf_counter(); sc.closest_point(x, abi.FILTER_DIRICHLET); ts.append(time.perf_counter() - t)
        print(f"{name} d/dmax [{lo:.3f},{hi:.3f}) frac {np.mean((d >= lo*dm)&(d < hi*dm)):.3f}  {min(ts)*1e3:8.2f} ms / {n} queries", flush=True)

which = sys.argv[1:] or ["2", "4", "5"]
if "2" in which:
    c = configs.config2()
    sc = B.Scene(c.vertices, c.segments, c.labels)
    p = np.random.default_rng(1).uniform(-1, 1, (4 << 20, 2))
    run("C2", sc, p)
if "4" in which:
    c = configs.config4(n_points=1 << 20)
    sc = B.Scene.mesh3(c.vertices, c.segments, c.labels)
    p = c.points[sc.inside(c.points).astype(bool)]
    run("C4", sc, p)
if "5" in which:
    c = configs.config5(n_points=1 << 21)
    tris, labels = configs.soup_shell(c)
    sc = B.Scene.mesh3(c.vertices, tris, labels)
    keep = np.zeros(len(c.points), bool)
    for m in configs.soup_components(c): keep |= m.inside(c.points)
    run("C5", sc, c.points[keep])
