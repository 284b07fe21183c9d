"""The library's sharded round (bvc_update_solution_sharded) against the
single-GPU round, bit for bit. Two ranks run as two processes on the one GPU of the
test box with a host-staged (gloo) all-gather communicator: nothing in the kernels
waits on another rank, only the host exchange does. One rank over NCCL exercises the
library's own ncclAllGather path."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEED = 11


def _problem(B, H, n_boundary):
    geom, pb = H.square_mixed()
    sc = B.Scene(*geom)
    region = B.SolveRegion(sc, offset=0.02, epsilon=1e-3 * sc.diagonal)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3 * sc.diagonal), nBoundary=n_boundary, nWalksNeumann=32,
                         nWalksDirichlet=64, offset=0.02)
    rng = np.random.default_rng(5)
    lo, hi = geom[0].min(0), geom[0].max(0)
    x = lo + (hi - lo) * rng.uniform(0.002, 0.998, (3001, 2))  # includes fallback-band points
    return sc, region, pb, cfg, x


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_boundary, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2302_11825_b200 as B
    from paper_2302_11825_b200 import distributed as D
    from tests import helpers as H

    sc, region, pb, cfg, x = _problem(B, H, n_boundary)
    b, e = D.shard_range(len(x), rank, world)
    pts = B.EvaluationPoints(x[b:e], 2, index_base=b)
    B.mark_evaluation_points(sc, region, cfg, pts)
    comm = D.host_staged_comm(B, dist, torch, rank, world)
    walks = 0
    for rnd in range(2):
        walks += B.update_solution_sharded(comm, sc, pb, region, cfg, pts, SEED, rnd, gradients=True)["cacheWalks"]
    state = {k: np.asarray(v) for k, v in pts.download().items()}
    # the host-buffer form of one round (bvc_update_solution_sharded_host)
    u, g = B.update_solution_sharded_host(comm, sc, pb, region, cfg, x[b:e], b, SEED, 7, gradients=True)
    state["host_u"], state["host_g"] = u, g
    q.put((rank, state, walks))
    dist.barrier()
    dist.destroy_process_group()


def _single(n_boundary):
    import paper_2302_11825_b200 as B
    from tests import helpers as H

    sc, region, pb, cfg, x = _problem(B, H, n_boundary)
    pts = B.EvaluationPoints(x, 2)
    B.mark_evaluation_points(sc, region, cfg, pts)
    walks = 0
    for rnd in range(2):
        walks += B.update_solution(sc, pb, region, cfg, pts, SEED, rnd, gradients=True)["cacheWalks"]
    state = dict(pts.download())
    state["host_u"], state["host_g"] = B.update_solution_host(sc, pb, region, cfg, x, SEED, 7, gradients=True)
    return state, walks, (sc, region, pb, cfg, x)


@pytest.mark.parametrize("n_boundary", [1024, 1001, 1])  # even, padded, and an empty shard
def test_two_rank_sharded_round_equals_single_gpu_round(n_boundary):
    import torch.multiprocessing as mp

    ref, ref_walks, _ = _single(n_boundary)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_boundary, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res.sort(key=lambda t: t[0])
    assert sum(t[2] for t in res) == ref_walks  # the shards' walks are the round's walks
    for k, v in ref.items():
        cat = np.concatenate([t[1][k] for t in res])
        assert np.array_equal(cat, np.asarray(v), equal_nan=True), k
    assert ref["fallback"].any() and (~ref["fallback"].astype(bool)).any()


def test_one_rank_nccl_sharded_round_equals_single_gpu_round():
    import paper_2302_11825_b200 as B

    ref, _, (sc, region, pb, cfg, x) = _single(1001)
    comm = B.Communicator.nccl(B.comm_unique_id(), 1, 0)
    pts = B.EvaluationPoints(x, 2)
    B.mark_evaluation_points(sc, region, cfg, pts)
    for rnd in range(2):
        B.update_solution_sharded(comm, sc, pb, region, cfg, pts, SEED, rnd, gradients=True)
    got = dict(pts.download())
    got["host_u"], got["host_g"] = B.update_solution_sharded_host(comm, sc, pb, region, cfg, x, 0, SEED, 7,
                                                                  gradients=True)
    for k, v in ref.items():
        assert np.array_equal(np.asarray(got[k]), np.asarray(v), equal_nan=True), k
