"""Projected strong scaling of the sharded round on one GPU: time rank 0's share of a
W-GPU round (its 1/W of the cache walks, a full-size cache assembled from copies of its
shard in place of the NCCL all-gather, its 1/W of the points, its fallback band) for
W = 1, 2, 4, 8 (the band walks overlap the shard's walks, as in bench.py's sharded round).
The all-gather itself (48 B x N over NVLink) is not included.
    python scripts/sim_rank.py [config [W ...]]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import ctypes as C  # noqa: E402

import paper_2302_11825_b200 as B  # noqa: E402
from paper_2302_11825_b200 import configs, distributed  # noqa: E402
from bench import build_problem  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
from paper_2302_11825_b200 import abi  # noqa: E402

c, scene, region = build_problem(cid, B, configs, abi)
cfg = c.cache
N = cfg.nBoundary
K = len(c.points)
res = {}
Ws = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
for W in Ws:
    pts = B.EvaluationPoints(c.points[: K // W], c.dim)
    B.mark_evaluation_points(scene, region, cfg, pts)
    spec = B.make_splat_config(scene, c.problem, cfg)

    marks = {}

    def tick(name):
        torch.cuda.synchronize()
        marks[name] = time.perf_counter()

    def step(rnd):
        tick("t0")
        s0, s1 = distributed.shard_range(N, 0, W)
        shard = B.generate_boundary_cache_with_fallback(scene, c.problem, region, cfg, c.seed, rnd, s0, s1, pts,
                                                        bool(c.gradients))
        tick("walks")
        ptr, nbytes = shard.packed()
        local = torch.as_tensor(distributed._DeviceBytes(ptr, nbytes), device="cuda")
        full = local.repeat(W)[: N * distributed.SAMPLE_BYTES // 4].contiguous()
        torch.cuda.synchronize()
        h = C.c_void_p()
        B.api._check(B.lib().bvc_boundary_cache_from_packed(C.c_void_p(full.data_ptr()), N, shard.dim, 0,
                                                            C.c_double(0.0), C.byref(h)))
        cache = B.BoundaryCache(h)
        tick("exchange")
        B.splat_range(cache, None, pts, spec, 0, 1 << 62, True, bool(c.gradients))
        tick("gather")

    for r in range(3):
        step(100 + r)
    ts = []
    for r in range(5):
        torch.cuda.synchronize()
        t = time.perf_counter()
        step(r)
        ts.append(time.perf_counter() - t)
    res[W] = float(np.median(ts))
    names = ["t0", "walks", "exchange", "gather"]
    print("   phases (ms):", {b: round((marks[b] - marks[a]) * 1e3, 3) for a, b in zip(names, names[1:])})
    eff = f", projected strong-scaling efficiency {res[1] / (W * res[W]):.3f}" if 1 in res else ""
    print(f"W={W}: rank-0 round {res[W] * 1e3:.3f} ms{eff}", flush=True)
