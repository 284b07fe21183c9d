"""bvc_update_solution_host (runSolveInMemory's round on host points, runner.cpp:116-169)
against the handle sequence it replaces (points_create, markEvaluationPoints,
updateSolution, solution()/gradient()): same u and grad u bit for bit, although the
points are uploaded and classified on a second stream while the cache walks run."""
import numpy as np
import pytest

import paper_2302_11825_b200 as B
from tests import helpers as H
from paper_2302_11825_b200 import abi, configs

pytestmark = pytest.mark.gpu


def _setup(cid, scale, n_points):
    c = configs.CONFIGS[cid](scale=scale)
    if c.extra.get("dim") == 3:
        sc = B.Scene.mesh3(c.vertices, c.segments, c.labels)
        region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
        x = c.points[sc.inside(c.points).astype(bool)][:n_points]
        return c, sc, region, x, 3
    sc = B.Scene(c.vertices, c.segments, c.labels)
    if c.region_mode == abi.REGION_SUBDOMAIN:
        sub = B.Scene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
        region = B.SolveRegion(sc, abi.REGION_SUBDOMAIN, c.region_offset, sub, epsilon=c.epsilon)
        x = c.points[region.boundary.inside(c.points).astype(bool)][:n_points]
    else:
        region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
        x = c.points[sc.inside(c.points).astype(bool)][:n_points]
    return c, sc, region, x, 2


@pytest.mark.parametrize("cid,scale", [(2, 1 / 32), (3, 1 / 128), (4, 1 / 256)])
def test_host_round_equals_handle_sequence(cid, scale):
    c, sc, region, x, dim = _setup(cid, scale, 20000)
    grads = bool(c.gradients)
    p = B.EvaluationPoints(x, dim)
    B.mark_evaluation_points(sc, region, c.cache, p)
    B.update_solution(sc, c.problem, region, c.cache, p, c.seed, 7, gradients=grads)
    ref = p.read_solution(gradient=grads)
    st = {}
    got = B.update_solution_host(sc, c.problem, region, c.cache, x, c.seed, 7, gradients=grads, stats=st)
    if grads:
        np.testing.assert_array_equal(got[0], ref[0])
        np.testing.assert_array_equal(got[1], ref[1])
    else:
        np.testing.assert_array_equal(got, ref)
    assert st["cacheWalks"] > 0 and np.all(np.isfinite(got[0] if grads else got))


def test_host_round_empty_and_errors():
    c, sc, region, x, dim = _setup(2, 1 / 64, 10)
    u = B.update_solution_host(sc, c.problem, region, c.cache, x[:0], c.seed, 1)
    assert u.shape == (0,)
    with pytest.raises(B.InvalidArgument):
        B.update_solution_host(sc, c.problem, region, c.cache, x, c.seed, 1, gradients=False,
                               out=(np.zeros(len(x)), np.zeros((len(x), 2))))


def test_overlapped_round_equals_sequential_pieces():
    """updateSolution runs the fallback-band walks on a second stream while the cache
    walks run; the reference's order (cache, splats, then band walks, cache.cpp:622-684)
    rebuilt from the separate entry points gives the same sums bit for bit."""
    c, sc, region, x, dim = _setup(2, 1 / 32, 20000)
    p = B.EvaluationPoints(x, dim)
    B.mark_evaluation_points(sc, region, c.cache, p)
    B.update_solution(sc, c.problem, region, c.cache, p, c.seed, 3, gradients=True)
    q = B.EvaluationPoints(x, dim)
    B.mark_evaluation_points(sc, region, c.cache, q)
    cache = B.generate_boundary_cache(sc, c.problem, region, c.cache, c.seed, 3)
    spec = B.make_splat_config(sc, c.problem, c.cache)
    B.splat_solution_gradient(cache, None, q, spec)
    B.fallback_walks(sc, c.problem, c.cache, q, c.seed, 3, True)
    a, b = p.download(), q.download()
    assert a["fallback"].sum() > 0
    for k in ("boundarySum", "boundaryGradSum", "nBoundary", "walkSum", "walkCount", "gradientWalkSum"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_shard_with_fallback_equals_separate_calls():
    """bvc_generate_boundary_cache_shard_fallback (a rank's shard plus its band walks on a
    second stream) against the shard and bvc_fallback_walks called one after the other."""
    c, sc, region, x, dim = _setup(2, 1 / 32, 20000)
    N = c.cache.nBoundary
    p = B.EvaluationPoints(x, dim)
    B.mark_evaluation_points(sc, region, c.cache, p)
    a = B.generate_boundary_cache_with_fallback(sc, c.problem, region, c.cache, c.seed, 5, N // 4, N // 2, p, True)
    q = B.EvaluationPoints(x, dim)
    B.mark_evaluation_points(sc, region, c.cache, q)
    b = B.generate_boundary_cache(sc, c.problem, region, c.cache, c.seed, 5, begin=N // 4, end=N // 2)
    B.fallback_walks(sc, c.problem, c.cache, q, c.seed, 5, True)
    ca, cb = a.download(), b.download()
    np.testing.assert_array_equal(ca["uHat"], cb["uHat"])
    np.testing.assert_array_equal(ca["dHat"], cb["dHat"])
    sa, sb = p.download(), q.download()
    assert sa["fallback"].sum() > 0
    for k in ("walkSum", "walkCount", "gradientWalkSum", "gradientWalkCount"):
        np.testing.assert_array_equal(sa[k], sb[k], err_msg=k)


def test_two_host_threads_run_rounds_concurrently():
    """Runtime state is per host thread and per device (capi.cu): two threads on their own
    streams run rounds at the same time and get exactly the sequential results."""
    import threading

    import torch

    geom, pb = H.square_mixed()
    sc = B.Scene(*geom)
    region = B.SolveRegion(sc, offset=0.02, epsilon=1e-3 * sc.diagonal)
    cfg = B.cache_config(nBoundary=2048, nWalksNeumann=32, nWalksDirichlet=64, offset=0.02)
    rng = np.random.default_rng(3)
    xs = [rng.uniform(0.01, 0.99, (4000, 2)) for _ in range(2)]

    def run(x, seed, out, key, stream=None, scene=None, reg=None):
        scene, reg = scene or sc, reg or region
        if stream is not None:
            B.set_stream(stream.cuda_stream)
        p = B.EvaluationPoints(x)
        B.mark_evaluation_points(scene, reg, cfg, p)
        for r in range(2):
            B.update_solution(scene, pb, reg, cfg, p, seed, r, gradients=True)
        out[key] = p.download()
        if stream is not None:
            B.synchronize()
            B.set_stream(None)

    seq = {}
    for k in range(2):
        run(xs[k], 100 + k, seq, k)
    # a fresh scene and region: both threads race for its lazy device state (upload, hint grid)
    sc2 = B.Scene(*geom)
    region2 = B.SolveRegion(sc2, offset=0.02, epsilon=1e-3 * sc2.diagonal)
    par = {}
    streams = [torch.cuda.Stream() for _ in range(2)]
    th = [threading.Thread(target=run, args=(xs[k], 100 + k, par, k, streams[k], sc2, region2)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for k in range(2):
        for name, v in seq[k].items():
            assert np.array_equal(np.asarray(par[k][name]), np.asarray(v), equal_nan=True), (k, name)


def test_a_waiting_round_does_not_block_another_threads_launches(monkeypatch):
    """A cache generation waits on the host for its failed-sample count. That read goes
    through pinned memory (read_device_int, capi.cu): a copy into pageable memory blocks inside
    the driver, and launches from other host threads queue up behind it. While thread A's
    walks (held to one block per SM, so that they last) are running, a small library call from
    thread B on its own stream returns in a fraction of their time."""
    import threading
    import time

    import torch

    monkeypatch.setenv("BVC_WALK_OCC", "1")
    c, sc, region, x, dim = _setup(4, 1 / 4, 1000)
    B.generate_boundary_cache(sc, c.problem, region, c.cache, c.seed, 0)  # lazy scene state, warm-up
    t_ref = np.linspace(0.5, 4.0, 256)
    B.eval_bessel(0, t_ref)
    res = {}

    def walks():
        B.set_stream(sa.cuda_stream)
        t0 = time.perf_counter()
        B.generate_boundary_cache(sc, c.problem, region, c.cache, c.seed, 1)
        B.synchronize()
        res["walks"] = time.perf_counter() - t0
        B.set_stream(None)

    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    th = threading.Thread(target=walks)
    torch.cuda.synchronize()
    th.start()
    time.sleep(0.05)
    B.set_stream(sb.cuda_stream)
    t0 = time.perf_counter()
    for _ in range(3):
        B.eval_bessel(0, t_ref)
    B.synchronize()
    small = time.perf_counter() - t0
    B.set_stream(None)
    th.join()
    assert res["walks"] > 0.15, res  # long enough for the comparison to mean something
    assert small < 0.3 * res["walks"], (small, res)


@pytest.mark.parametrize("cid,scale", [(1, 1 / 16), (4, 1 / 256)])
def test_last_round_kernel_seconds_bracket_the_hot_launches(cid, scale):
    """bvc_last_round_kernel_seconds: the round's main walk and gather launches, each
    inside its phase (generateSeconds / splatSeconds), reset by a round without them"""
    c, sc, region, x, dim = _setup(cid, scale, 4000)
    p = B.EvaluationPoints(x, dim)
    B.mark_evaluation_points(sc, region, c.cache, p)
    st = B.update_solution(sc, c.problem, region, c.cache, p, c.seed, 3, gradients=bool(c.gradients))
    k = B.last_round_kernel_seconds()
    assert 0.0 < k["walk"] <= st["generateSeconds"] * 1.001
    assert 0.0 < k["gather"] <= st["splatSeconds"] * 1.001
    empty = B.EvaluationPoints(x[:0], dim)
    B.update_solution(sc, c.problem, region, c.cache, empty, c.seed, 4)
    k2 = B.last_round_kernel_seconds()
    assert k2["walk"] > 0.0 and k2["gather"] == 0.0  # no points: no gather launch
