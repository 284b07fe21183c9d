"""Edge cases of the drop-in boundary: empty and single-element inputs, all points in
the fallback band, caches without samples, points sitting on samples, accumulation
across calls, and the reference's input validation (cache.cpp / pointwise.cpp)."""
import numpy as np
import pytest

import paper_2302_11825_b200 as B
from oracle import oracle as O
from paper_2302_11825_b200 import abi
from tests import helpers as H

pytestmark = pytest.mark.gpu


def _disk():
    geom, pb = H.disk_linear()
    sc = B.Scene(*geom)
    region = B.SolveRegion(sc, offset=0.05, epsilon=1e-3)
    return geom, pb, sc, region


def test_empty_point_sets_and_empty_caches():
    geom, pb, sc, region = _disk()
    cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=64, nWalksNeumann=8, nWalksDirichlet=16, offset=0.05)
    empty = B.EvaluationPoints(np.zeros((0, 2)))
    B.mark_evaluation_points(sc, region, cfg, empty)
    st = B.update_solution(sc, pb, region, cfg, empty, 1, 0, gradients=True)
    assert st["cacheWalks"] > 0 and empty.download()["boundarySum"].shape == (0,)
    u = empty.read_solution(gradient=False)
    assert u.shape == (0,)
    # a cache with one sample, a source cache with none
    one = B.BoundaryCache.from_arrays([[1.0, 0.0]], [[1.0, 0.0]], [1.0], [2.0], [0.5])
    p = B.EvaluationPoints([[0.0, 0.0], [0.5, 0.1]])
    spec = abi.SplatConfig(H.kspec(0, 0, 2, sc.diagonal), 1e-12 * sc.diagonal, 0, 0)
    B.splat_solution_gradient(one, None, p, spec)
    s = p.download()
    assert np.all(s["nBoundary"] == 1) and np.all(s["mSource"] == 0)
    ref = O.oracle_splat(H.kspec(0, 0, 2, sc.diagonal), 1e-12 * sc.diagonal,
                         dict(z=np.array([[1.0, 0.0]]), n=np.array([[1.0, 0.0]]), pdf=np.ones(1), uHat=[2.0],
                              dHat=[0.5], weight=np.zeros(1)), None, [[0.0, 0.0], [0.5, 0.1]], value=True,
                         gradient=True)
    assert H.rel_err(s["boundarySum"], ref["boundarySum"]) < 1e-5
    assert H.rel_err(s["boundaryGradSum"], ref["boundaryGradSum"]) < 1e-5


def test_all_points_in_the_fallback_band():
    geom, pb, sc, region = _disk()
    cfg = B.cache_config(B.walk_config(epsilon=1e-3, nWalks=256), nBoundary=64, nWalksNeumann=8,
                         nWalksDirichlet=16, offset=0.05)
    th = np.linspace(0, 2 * np.pi, 50, endpoint=False)
    x = 0.98 * np.stack([np.cos(th), np.sin(th)], 1)  # within l = 0.05 of the Dirichlet circle
    p = B.EvaluationPoints(x)
    B.mark_evaluation_points(sc, region, cfg, p)
    assert p.download()["fallback"].all()
    B.update_solution(sc, pb, region, cfg, p, 3, 0, gradients=True)
    s = p.download()
    assert np.all(s["nBoundary"] == 0) and np.all(s["walkCount"] == 256)
    u = p.solution(s)
    assert np.max(np.abs(u - x[:, 0])) < 0.05  # u = x, plain walks with 256 samples


def test_points_on_samples_and_accumulation_across_calls():
    geom, pb, sc, region = _disk()
    rng = np.random.default_rng(4)
    z = rng.normal(size=(300, 2))
    z /= np.linalg.norm(z, axis=1)[:, None]
    bc = B.BoundaryCache.from_arrays(z, z, np.full(300, 1 / (2 * np.pi)), z[:, 0], z[:, 0])
    spec = abi.SplatConfig(H.kspec(0, 0, 2, sc.diagonal), 1e-12 * sc.diagonal, 0, 0)
    x = np.concatenate([z[:5], rng.uniform(-0.5, 0.5, (20, 2))])
    p = B.EvaluationPoints(x)
    B.splat_solution_gradient(bc, None, p, spec)
    s1 = p.download()
    assert np.all(s1["skipped"][:5] == 2) and np.all(s1["skipped"][5:] == 0)  # value + gradient passes
    assert np.all(s1["nBoundary"][:5] == 299) and np.all(np.isfinite(s1["boundarySum"]))
    B.splat_solution_gradient(bc, None, p, spec)
    s2 = p.download()
    np.testing.assert_array_equal(s2["boundarySum"], 2 * s1["boundarySum"])  # splats accumulate (x2 exact)
    assert np.all(s2["nBoundary"] == 2 * s1["nBoundary"])
    p.reset()
    assert np.all(p.download()["nBoundary"] == 0)


def test_reference_input_validation():
    geom, pb, sc, region = _disk()
    cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=16, nWalksNeumann=4, nWalksDirichlet=4, offset=0.05)
    # r_min above epsilon (pointwise.h:39-44)
    bad = B.cache_config(B.walk_config(epsilon=1e-3, rMin=1e-2), nBoundary=16, offset=0.05)
    with pytest.raises(B.InvalidArgument):
        B.generate_boundary_cache(sc, pb, region, bad, 1, 0)
    # kernel spec: sigma = 0 iff Poisson (kernels.h:32-37)
    badk = H.make_problem(H.kspec(0, 1.0), g=pb.g)
    with pytest.raises(B.InvalidArgument):
        B.update_solution(sc, badk, region, cfg, B.EvaluationPoints([[0.0, 0.0]]), 1, 0)
    # a scene without Dirichlet boundary cannot terminate walks (pointwise.cpp:217-218)
    v, s, _ = O.rectangle_geometry([0, 0], [1, 1], [1, 1, 1, 1])
    neu = B.Scene(v, s, [1, 1, 1, 1])
    with pytest.raises(B.SolverError):
        B.wost_solve(neu, pb, [[0.5, 0.5]], B.walk_config(nWalks=4))
    # dimension mismatch between points and kernel
    spec3 = abi.SplatConfig(H.kspec(0, 0, 3, 1.0), 1e-12, 0, 0)
    one = B.BoundaryCache.from_arrays([[1.0, 0.0]], [[1.0, 0.0]], [1.0], [2.0], [0.5])
    with pytest.raises(B.InvalidArgument):
        B.splat_solution(one, None, B.EvaluationPoints([[0.0, 0.0]]), spec3)


def test_large_point_count_bitwise_shard_invariance():
    """1M points split into uneven ranges: bitwise the same sums as one call."""
    geom, pb, sc, region = _disk()
    rng = np.random.default_rng(9)
    z = rng.normal(size=(2048, 2))
    z /= np.linalg.norm(z, axis=1)[:, None]
    bc = B.BoundaryCache.from_arrays(z, z, np.full(2048, 1 / (2 * np.pi)), z[:, 1], z[:, 0])
    spec = abi.SplatConfig(H.kspec(0, 0, 2, sc.diagonal), 1e-12 * sc.diagonal, 0, 0)
    x = rng.uniform(-0.7, 0.7, (1 << 20, 2))
    a = B.EvaluationPoints(x)
    B.splat_solution_gradient(bc, None, a, spec)
    b = B.EvaluationPoints(x)
    cuts = [0, 1, 4097, 300000, 777777, 1 << 20]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        B.splat_range(bc, None, b, spec, lo, hi, True, True)
    sa, sb = a.download(), b.download()
    assert np.array_equal(sa["boundarySum"], sb["boundarySum"])
    assert np.array_equal(sa["boundaryGradSum"], sb["boundaryGradSum"])
