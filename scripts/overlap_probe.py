"""Co-residency probe (C5 shapes): how long the round-r gather and the round-(r+1) cache
walks take alone, with capped occupancy, and running concurrently on two streams from
two host threads. Decides whether pipelining rounds (walks of r+1 under the gather of r)
pays. Usage: python scripts/overlap_probe.py [n_points] [cfg]"""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import abi, configs  # noqa: E402

n_points = int(sys.argv[1]) if len(sys.argv) > 1 else 4_194_304
cfg_id = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if cfg_id == 5:
    configs.CONFIGS[5] = lambda: configs.config5(n_points=n_points)
c, scene, region = bench.build_problem(cfg_id, B, configs, abi)
cfg = c.cache
pts = B.EvaluationPoints(c.points, c.dim)
B.mark_evaluation_points(scene, region, cfg, pts)
spec = B.make_splat_config(scene, c.problem, cfg)
cache0 = B.generate_boundary_cache(scene, c.problem, region, cfg, c.seed, 0)
torch.cuda.synchronize()
print("points", len(c.points), flush=True)


def t_gather():
    torch.cuda.synchronize()
    t = time.perf_counter()
    B.splat_range(cache0, None, pts, spec, 0, 1 << 62, True, bool(c.gradients))
    B.synchronize()
    return time.perf_counter() - t


def t_walks(r=1):
    torch.cuda.synchronize()
    t = time.perf_counter()
    cc = B.generate_boundary_cache(scene, c.problem, region, cfg, c.seed, r)
    B.synchronize()
    dt = time.perf_counter() - t
    del cc
    return dt


def setenv(k, v):
    if v is None:
        os.environ.pop(k, None)
    else:
        os.environ[k] = str(v)


t_gather(); t_walks()
for occ in [None, 1, 2, 3]:
    setenv("BVC_GATHER_OCC", occ)
    print("gather alone occ", occ, round(t_gather(), 3), flush=True)
setenv("BVC_GATHER_OCC", None)
for occ in [None, 2, 4, 6]:
    setenv("BVC_WALK_OCC", occ)
    print("walks alone occ", occ, round(t_walks(), 3), flush=True)
setenv("BVC_WALK_OCC", None)

hi = torch.cuda.Stream(priority=-1)
lo = torch.cuda.Stream(priority=0)


def concurrent(gocc, wocc, walk_hi=True):
    setenv("BVC_GATHER_OCC", gocc)
    setenv("BVC_WALK_OCC", wocc)
    res = {}

    def g():
        B.set_stream((lo if walk_hi else hi).cuda_stream)
        t = time.perf_counter()
        B.splat_range(cache0, None, pts, spec, 0, 1 << 62, True, bool(c.gradients))
        B.synchronize()
        res["g"] = time.perf_counter() - t

    def w():
        B.set_stream((hi if walk_hi else lo).cuda_stream)
        t = time.perf_counter()
        cc = B.generate_boundary_cache(scene, c.problem, region, cfg, c.seed, 1)
        B.synchronize()
        res["w"] = time.perf_counter() - t
        del cc

    torch.cuda.synchronize()
    t = time.perf_counter()
    th = [threading.Thread(target=g), threading.Thread(target=w)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    torch.cuda.synchronize()
    res["total"] = time.perf_counter() - t
    return {k: round(v, 3) for k, v in res.items()}


for gocc, wocc in [(None, None), (1, None), (2, None), (3, None), (2, 4), (1, 6), (3, 2)]:
    print("concurrent gather occ", gocc, "walk occ", wocc, concurrent(gocc, wocc), flush=True)
print("concurrent gather-high-priority", concurrent(2, None, walk_hi=False), flush=True)
