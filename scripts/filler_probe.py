"""Filler probe (C5 shapes): the gather at full occupancy with the cache walks of another
part of the samples co-resident at 1-2 blocks per SM (launched first). Reports each
kernel's time alone and together. Usage: python scripts/filler_probe.py [n_points] [frac]"""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402

n_points = int(sys.argv[1]) if len(sys.argv) > 1 else 8_388_608
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
configs.CONFIGS[5] = lambda: configs.config5(n_points=n_points)
c, scene, region = bench.build_problem(5, B, configs, abi)
cfg = c.cache
N = int(cfg.nBoundary)
pts = B.EvaluationPoints(c.points, c.dim)
B.mark_evaluation_points(scene, region, cfg, pts)
spec = B.make_splat_config(scene, c.problem, cfg)
cache0 = B.generate_boundary_cache(scene, c.problem, region, cfg, c.seed, 0)
torch.cuda.synchronize()
print("points", len(c.points), "samples", N, "walk part", frac, flush=True)


def setenv(k, v):
    if v is None:
        os.environ.pop(k, None)
    else:
        os.environ[k] = str(v)


def gather():
    t = time.perf_counter()
    B.splat_range(cache0, None, pts, spec, 0, 1 << 62, True, False)
    B.synchronize()
    return time.perf_counter() - t


def walks(r=1):
    t = time.perf_counter()
    cc = B.generate_boundary_cache(scene, c.problem, region, cfg, c.seed, r, begin=0, end=int(N * frac))
    B.synchronize()
    dt = time.perf_counter() - t
    del cc
    return dt


gather(); walks()
g0 = min(gather() for _ in range(2))
print("gather alone", round(g0, 3), flush=True)
w_alone = {}
for occ in [None, 1, 2, 3]:
    setenv("BVC_WALK_OCC", occ)
    w_alone[occ] = walks()
    print("walks alone occ", occ, round(w_alone[occ], 3), flush=True)
setenv("BVC_WALK_OCC", None)

s_w = torch.cuda.Stream(priority=-1)
s_g = torch.cuda.Stream(priority=0)


import queue  # noqa: E402


class Worker(threading.Thread):
    """A long-lived host thread with its own library stream and warmed-up workspaces."""

    def __init__(self, stream, fn):
        super().__init__(daemon=True)
        self.stream, self.fn = stream, fn
        self.q, self.out = queue.Queue(), queue.Queue()
        self.start()

    def run(self):
        B.set_stream(self.stream.cuda_stream)
        while True:
            self.q.get()
            t0 = time.perf_counter()
            dt = self.fn()
            self.out.put((t0, dt))


W_w, W_g = Worker(s_w, walks), Worker(s_g, gather)
for w in (W_w, W_g):  # warm-up: allocations of this thread's workspaces
    w.q.put(1); w.out.get()
    w.q.put(1); w.out.get()


def together(wocc, gocc=None, delay=0.05):
    setenv("BVC_WALK_OCC", wocc)
    setenv("BVC_GATHER_OCC", gocc)
    torch.cuda.synchronize()
    t = time.perf_counter()
    W_w.q.put(1)
    time.sleep(delay)
    W_g.q.put(1)
    tw0, w = W_w.out.get()
    tg0, g = W_g.out.get()
    torch.cuda.synchronize()
    res = {"w": w, "g": g, "g_start": tg0 - t, "total": time.perf_counter() - t, "sequential": g0 + w_alone[None]}
    setenv("BVC_WALK_OCC", None)
    setenv("BVC_GATHER_OCC", None)
    return {k: round(v, 3) for k, v in res.items()}


for carve in [None, 44]:
    setenv("BVC_WALK_CARVEOUT", carve)
    setenv("BVC_GATHER_CARVEOUT", carve)
    g1 = gather()
    setenv("BVC_WALK_OCC", None)
    w1 = walks()
    print("carve-out", carve, "gather alone", round(g1, 3), "walks alone", round(w1, 3), flush=True)
    for wocc, gocc in [(1, None), (2, None), (3, None), (2, 3)]:
        print("  together walk occ", wocc, "gather occ", gocc, together(wocc, gocc), flush=True)
