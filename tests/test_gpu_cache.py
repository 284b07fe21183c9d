"""Cache construction (generateBoundaryCache cache.cpp:301-390, generateSourceCache
392-406) and one progressive round (updateSolution 622-684) on the GPU."""
import numpy as np
import pytest

import paper_2302_11825_b200 as B
from oracle import oracle as O
from paper_2302_11825_b200 import abi, configs
from tests import helpers as H

pytestmark = pytest.mark.gpu


def _setup(maker, offset=0.05):
    geom, pb = maker()
    sc = B.Scene(*geom)
    region = B.SolveRegion(sc, offset=offset, epsilon=1e-3)
    return geom, pb, sc, region


def test_pdfs_reflecting_data_and_walk_accounting():
    """test_cache.cpp:262-293."""
    geom, pb, sc, region = _setup(H.square_mixed)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=96, nWalksNeumann=8, nWalksDirichlet=16, offset=0.05)
    st = {}
    cache = B.generate_boundary_cache(sc, pb, region, cfg, 11, 0, stats=st)
    c = cache.download()
    assert cache.n == 96
    length = O.OracleScene(region.vertices, region.segments, region.labels).diagonal  # noqa: F841
    L = np.sum(np.linalg.norm(region.vertices[region.segments[:, 1]] - region.vertices[region.segments[:, 0]], axis=1))
    np.testing.assert_allclose(c["pdf"], 1.0 / L, rtol=1e-6)
    kinds = region.kinds[c["segment"]]
    neu = kinds == abi.SEG_KNOWN_NEUMANN
    assert neu.sum() > 0 and np.all(c["dHat"][neu] == 0.0)
    assert np.all(np.isfinite(c["uHat"])) and np.all(np.isfinite(c["dHat"]))
    if st["resampled"] == 0:
        assert st["cacheWalks"] == 96 * (8 + 16) - neu.sum() * 16
    assert st["cacheSteps"] > st["cacheWalks"]


def test_positions_are_stratified_like_the_reference():
    """BoundarySampler::sample with stratification: sample k lies in stratum k (sampling.cpp:37-44)."""
    geom, pb, sc, region = _setup(H.disk_linear)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=1000, nWalksNeumann=1, nWalksDirichlet=1, offset=0.05)
    c = B.generate_boundary_cache(sc, pb, region, cfg, 3, 0).download()
    L = np.sum(np.linalg.norm(region.vertices[region.segments[:, 1]] - region.vertices[region.segments[:, 0]], axis=1))
    u = c["arc"] / L  # single loop: arc-length fraction
    k = np.arange(1000)
    assert np.all(u >= k / 1000 - 1e-6) and np.all(u <= (k + 1) / 1000 + 1e-6)


def test_offset_disk_closed_form():
    """test_cache.cpp:295-319: disk-poisson estimates vs the radial solution."""
    geom, pb, sc, region = _setup(H.disk_poisson)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=512, nWalksNeumann=64, nWalksDirichlet=640,
                         offset=0.05)
    c = B.generate_boundary_cache(sc, pb, region, cfg, 13, 0).download()
    z, n = c["z"], c["n"]
    du = c["uHat"] - 0.25 * (np.sum(z * z, 1) - 1)
    dd = c["dHat"] - 0.5 * np.sum(z * n, 1)
    assert abs(du.mean()) <= 4 * du.std(ddof=1) / np.sqrt(len(du))
    assert abs(dd.mean()) <= 4 * dd.std(ddof=1) / np.sqrt(len(dd))
    assert abs(c["dHat"].mean() - (1 - 0.05) / 2) <= max(4 * c["dHat"].std(ddof=1) / np.sqrt(len(dd)), 5e-3)


def test_cache_vs_reference_estimates_at_same_positions():
    """Per-sample z-test of the GPU cache against the reference's wostSolve /
    wostNormalDerivative at the GPU's own sample positions."""
    geom, pb, sc, region = _setup(H.square_mixed)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=48, nWalksNeumann=4096, nWalksDirichlet=4096,
                         offset=0.05)
    c = B.generate_boundary_cache(sc, pb, region, cfg, 17, 0).download()
    rs = O.RefScene(*geom)
    kinds = region.kinds[c["segment"]]
    wc = abi.default_walk_config()
    wc.nWalks, wc.epsilon = 4096, 1e-3
    # GPU per-sample standard errors from independent re-estimates at the same positions
    x_u = np.where((kinds == abi.SEG_KNOWN_NEUMANN)[:, None], c["z"] - 0.5e-3 * c["n"], c["z"])
    gu = B.wost_solve(sc, pb, x_u, B.walk_config(epsilon=1e-3, nWalks=4096, seed=99))
    zs = []
    for i in range(len(c["pdf"])):
        wc.seed = 1000 + i
        r = rs.solve(pb, x_u[i], wc, 1)
        zs.append(H.zscore(c["uHat"][i], gu["se"][i], r[0], r[1]))
    zs = np.abs(np.array(zs))
    assert np.sum(zs > 3) <= 2, zs


def test_shard_union_equals_full_cache():
    """RNG keyed by global sample index: shards [0,a) + [a,N) reproduce the full cache bitwise."""
    geom, pb, sc, region = _setup(H.square_mixed)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=256, nWalksNeumann=16, nWalksDirichlet=32,
                         offset=0.05)
    full = B.generate_boundary_cache(sc, pb, region, cfg, 5, 2).download()
    a = B.generate_boundary_cache(sc, pb, region, cfg, 5, 2, begin=0, end=100).download()
    b = B.generate_boundary_cache(sc, pb, region, cfg, 5, 2, begin=100, end=256).download()
    for key in ("z", "uHat", "dHat", "pdf"):
        assert np.array_equal(np.concatenate([a[key], b[key]]), full[key]), key
    other = B.generate_boundary_cache(sc, pb, region, cfg, 5, 3).download()
    assert not np.array_equal(other["uHat"], full["uHat"])


def test_allgathered_shards_with_voronoi_weights_match_the_full_cache():
    """The multi-GPU exchange (distributed.generate_and_allgather) on one device: packed
    shards concatenated in order, then assignVoronoiWeights over the whole round."""
    import torch

    from paper_2302_11825_b200 import distributed

    geom, pb, sc, region = _setup(H.disk_linear)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=300, nWalksNeumann=8, nWalksDirichlet=16,
                         offset=0.05, voronoi=1)
    full = B.generate_boundary_cache(sc, pb, region, cfg, 8, 1).download()
    assert abs(full["weight"].sum() - np.sum(np.linalg.norm(
        region.vertices[region.segments[:, 1]] - region.vertices[region.segments[:, 0]], axis=1))) < 1e-4
    parts = []
    for r in range(3):
        lo, hi = distributed.shard_range(300, r, 3)
        shard = B.generate_boundary_cache(sc, pb, region, cfg, 8, 1, begin=lo, end=hi)
        ptr, nbytes = shard.packed()
        parts.append(torch.as_tensor(distributed._DeviceBytes(ptr, nbytes), device="cuda").clone())
        del shard
    joined = torch.cat(parts)
    torch.cuda.synchronize()
    import ctypes as C
    h = C.c_void_p()
    B.api._check(B.lib().bvc_boundary_cache_from_packed(C.c_void_p(joined.data_ptr()), 300, 2, 0, C.c_double(0.0),
                                                        C.byref(h)))
    cache = B.BoundaryCache(h)
    cache.assign_voronoi(region)
    got = cache.download()
    for key in ("z", "n", "uHat", "dHat", "pdf", "weight", "arc"):
        assert np.array_equal(got[key], full[key]), key


def test_source_cache_fields():
    """test_cache.cpp:363-379."""
    geom, pb, sc, region = _setup(H.disk_poisson)
    cfg = B.cache_config(nSource=200)
    s = B.generate_source_cache(pb, region, cfg, 23, 0)
    d = s.download()
    assert s.m == 200
    np.testing.assert_allclose(d["pdf"], 1.0 / region.area, rtol=1e-6)
    assert np.all(d["f"] == 1.0)
    assert np.all(region.boundary.inside(d["y"]))
    geom, pbl, scl, rl = _setup(H.disk_linear)
    assert B.generate_source_cache(pbl, rl, cfg, 23, 0).m == 0


def test_update_solution_rounds_accumulate_and_commute():
    """test_cache.cpp:571-621."""
    geom, pb, sc, region = _setup(H.disk_poisson)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3, nWalks=64), nBoundary=48, nSource=48, nWalksNeumann=4,
                         nWalksDirichlet=8, offset=0.05)
    pts = B.EvaluationPoints([[0, 0], [0.3, 0.2], [0.97, 0]])
    B.mark_evaluation_points(sc, region, cfg, pts)
    st = pts.download()
    assert not st["fallback"][0] and st["fallback"][2]
    B.update_solution(sc, pb, region, cfg, pts, 41, 0)
    B.update_solution(sc, pb, region, cfg, pts, 41, 1)
    st = pts.download()
    assert st["nBoundary"][0] == 96 and st["mSource"][0] == 96 and st["walkCount"][2] == 128
    fwd, rev = B.EvaluationPoints([[0.3, 0.2]]), B.EvaluationPoints([[0.3, 0.2]])
    for p in (fwd, rev):
        B.mark_evaluation_points(sc, region, cfg, p)
    B.update_solution(sc, pb, region, cfg, fwd, 43, 0)
    B.update_solution(sc, pb, region, cfg, fwd, 43, 1)
    B.update_solution(sc, pb, region, cfg, rev, 43, 1)
    B.update_solution(sc, pb, region, cfg, rev, 43, 0)
    f, r = fwd.download(), rev.download()
    assert f["boundarySum"][0] == r["boundarySum"][0] and f["sourceSum"][0] == r["sourceSum"][0]


@pytest.mark.ref
def test_mark_points_match_reference():
    geom, pb, sc, region = _setup(H.disk_poisson)
    rs = O.RefScene(*geom)
    rr = O.RefRegion(rs, abi.REGION_WHOLE_DOMAIN, 0.05, eps=1e-3)
    cfg = B.cache_config(offset=0.05)
    rng = np.random.default_rng(2)
    r = np.sqrt(rng.uniform(0, 0.99, 4000))
    a = rng.uniform(0, 2 * np.pi, 4000)
    x = np.stack([r * np.cos(a), r * np.sin(a)], 1)
    pts = B.EvaluationPoints(x)
    B.mark_evaluation_points(sc, region, cfg, pts)
    st = pts.download()
    fb, gu = O.ref_mark_points(rs, rr, cfg, x)
    assert np.mean(st["fallback"] == fb) > 0.999 and np.mean(st["gradientUnreliable"] == gu) > 0.999


def test_end_to_end_config2_small_vs_exact_and_reference():
    """A reduced C2 round (u = x exactly): GPU and reference errors have the same scale."""
    c = configs.config2(scale=1 / 16, grid_n=64)
    sc = B.Scene(c.vertices, c.segments, c.labels)
    region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
    c.cache.nWalksNeumann = c.cache.nWalksDirichlet = 64
    c.cache.walk.nWalks = 64
    pts = B.EvaluationPoints(c.points)
    B.mark_evaluation_points(sc, region, c.cache, pts)
    B.update_solution(sc, c.problem, region, c.cache, pts, c.seed, 0, gradients=True)
    st = pts.download()
    u = pts.solution(st)
    assert np.all(np.isfinite(u))
    err_gpu = np.sqrt(np.mean((u - c.points[:, 0]) ** 2))
    rs = O.RefScene(c.vertices, c.segments, c.labels)
    rr = O.RefRegion(rs, abi.REGION_WHOLE_DOMAIN, c.region_offset, eps=c.epsilon)
    cfg = c.cache
    cfg.threads = 0
    ref = O.ref_update_solution(rs, c.problem, rr, cfg, c.points, c.seed, 0, gradients=False)
    err_ref = np.sqrt(np.mean((ref["u"] - c.points[:, 0]) ** 2))
    assert err_gpu < 2.0 * err_ref + 0.01, (err_gpu, err_ref)
    assert np.array_equal(st["fallback"], ref["fallback"])
