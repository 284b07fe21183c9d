"""Projected strong scaling of the library's sharded round on one GPU: rank 0 of W runs
bvc_update_solution_sharded on its 1/W of the samples and points, through a communicator
whose all-gather replicates rank 0's shard W times on the device (standing in for the
NCCL all-gather of 48 B x N over NVLink, whose own time is not included). Prints rank 0's
round time per W and the implied efficiency.
    python scripts/sim_rank.py [config [W ...]]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_11825_b200 as B  # noqa: E402
from bench import build_problem  # noqa: E402
from paper_2302_11825_b200 import abi, configs, distributed  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
Ws = [int(a) for a in sys.argv[2:]] or [1, 2, 4, 8]
c, scene, region = build_problem(cid, B, configs, abi)
cfg = c.cache
K = len(c.points)
res = {}
for W in Ws:
    def fn(send, recv, nbytes, W=W):
        dev = torch.device("cuda", torch.cuda.current_device())
        src = torch.as_tensor(distributed._DeviceBytes(send, nbytes), device=dev)
        dst = torch.as_tensor(distributed._DeviceBytes(recv, nbytes * W), device=dev)
        dst.view(W, -1).copy_(src.view(1, -1).expand(W, -1))
        torch.cuda.synchronize()

    comm = B.Communicator.from_allgather(W, 0, fn)
    b, e = distributed.shard_range(K, 0, W)
    pts = B.EvaluationPoints(c.points[b:e], c.dim, index_base=b)
    B.mark_evaluation_points(scene, region, cfg, pts)
    times = []
    for rnd in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        B.update_solution_sharded(comm, scene, c.problem, region, cfg, pts, c.seed, rnd, gradients=bool(c.gradients))
        e1.record()
        torch.cuda.synchronize()
        if rnd >= 3:
            times.append(e0.elapsed_time(e1))
    res[W] = float(np.median(times))
    del comm
t1 = res.get(1, res[Ws[0]] * Ws[0])
print(json.dumps({"config": cid, "rank0_round_ms": res,
                  "projected_efficiency": {W: t1 / (W * t) for W, t in res.items()},
                  "note": "rank 0 of W on one GPU; the all-gather is a device-side replication (NVLink time excluded)"}))
