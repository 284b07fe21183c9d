"""Multi-rank plumbing on CPU (gloo, world_size 2): shard arithmetic, the cache
all-gather of packed 48-byte samples, and the point-range gather — the parts of the
N>1 path that do not need a GPU. The compute stand-in is the oracle
(test infrastructure), which makes the rank decomposition checkable exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2302_11825_b200 import distributed as D


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 16384, 1048576):
        for w in (1, 2, 3, 8):
            ranges = [D.shard_range(n, r, w) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            assert max(D.shard_sizes(n, w)) - min(D.shard_sizes(n, w)) <= 1
    with pytest.raises(ValueError):
        D.shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from tests import helpers as H

    N = 101
    rng = np.random.default_rng(7)
    # every rank builds the same synthetic "global" cache; rank r contributes its shard as bytes
    zz = rng.normal(size=(N, 2))
    full = np.zeros((N, 12), np.float32)
    full[:, 0:2] = zz
    full[:, 3:5] = zz / np.linalg.norm(zz, axis=1)[:, None]
    full[:, 6] = 0.1
    full[:, 7] = rng.uniform(-1, 1, N)
    full[:, 8] = rng.uniform(-1, 1, N)
    s0, s1 = D.shard_range(N, rank, world)
    local = torch.from_numpy(full[s0:s1].copy().view(np.int32).ravel())
    sizes = [s * D.SAMPLE_BYTES for s in D.shard_sizes(N, world)]

    class _Dist:
        all_gather = staticmethod(dist.all_gather)

    gathered = D.allgather_bytes(_Dist, torch, local, sizes).numpy().view(np.float32).reshape(N, 12)
    ok_cache = bool(np.array_equal(gathered, full))
    # point sharding: each rank splats its contiguous range; the union equals the full splat
    x = rng.uniform(-0.5, 0.5, (50, 2))
    p0, p1 = D.shard_range(len(x), rank, world)
    cache = dict(z=gathered[:, 0:2].astype(float), n=gathered[:, 3:5].astype(float), pdf=gathered[:, 6].astype(float),
                 uHat=gathered[:, 7].astype(float), dHat=gathered[:, 8].astype(float), weight=np.zeros(N))
    spec = H.kspec(0, 0, 2, 4.0)
    mine = O.oracle_splat(spec, 1e-12 * 4.0, cache, None, x[p0:p1], value=True)["boundarySum"]
    parts = [None] * world
    dist.all_gather_object(parts, (p0, mine.tolist()))
    ref = O.oracle_splat(spec, 1e-12 * 4.0, cache, None, x, value=True)["boundarySum"]
    got = np.zeros(len(x))
    for a, vals in parts:
        got[a:a + len(vals)] = vals
    out[rank] = (ok_cache, bool(np.array_equal(got, ref)))
    dist.destroy_process_group()


def test_gloo_world2_cache_allgather_and_point_shards():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res == {0: (True, True), 1: (True, True)}


def test_library_shard_layout_matches_the_python_ranges():
    """bvc_shard_layout (host arithmetic of the library's sharded round): contiguous
    balanced ranges, and the all-gather's padded per-rank count ceil(n / W)."""
    import paper_2302_11825_b200 as B

    for n in (1, 7, 1001, 16384, 1048576):
        for w in (1, 2, 3, 8):
            for r in range(w):
                b, e, cap = B.shard_layout(n, w, r)
                assert (b, e) == D.shard_range(n, r, w)
                assert cap == -(-n // w) and e - b <= cap
    with pytest.raises(B.BvcError):
        B.shard_layout(10, 2, 2)


def test_library_communicators_host_side():
    """bvc_comm handles without a device: a host-staged communicator is created, reports
    its ranks and is destroyed; invalid ranks are refused; the sharded round itself
    needs the GPU and says so (no CPU fallback)."""
    import paper_2302_11825_b200 as B

    calls = []
    comm = B.Communicator.from_allgather(4, 3, lambda s, r, n: calls.append(n))
    assert (comm.nranks, comm.rank) == (4, 3)
    del comm
    with pytest.raises(B.BvcError):
        B.Communicator.from_allgather(2, 2, lambda s, r, n: None)
    if torch.cuda.is_available():
        pytest.skip("no-device behaviour only")
    one = B.Communicator.from_allgather(1, 0, lambda s, r, n: None)
    geom = ([[0, 0], [1, 0], [1, 1], [0, 1]], [[0, 1], [1, 2], [2, 3], [3, 0]], [0, 0, 0, 0])
    sc = B.Scene(*geom)
    region = B.SolveRegion(sc, offset=0.05, epsilon=1e-3)
    pb = B.problem(B.poisson(2), g=B.field(B.abi.FIELD_LINEAR, 1.0, 0.0, 0.0, 0.0))
    with pytest.raises(B.NoDeviceError):
        B.update_solution_sharded_host(one, sc, pb, region, B.cache_config(), np.zeros((3, 2)) + 0.5, 0, 1, 0)
