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


def _region_from_loop(loop_geom):
    """a SolveRegion whose boundary is exactly `loop_geom` (a Subdomain loop inside a
    larger all-Dirichlet square), so the source sampler samples that loop's interior"""
    v, s, l = loop_geom
    lo, hi = v.min(0) - 0.5, v.max(0) + 0.5
    outer = O.rectangle_geometry(lo, hi, [0, 0, 0, 0])
    sc = B.Scene(*outer)
    sub = B.Scene(v, s, np.zeros(len(s), np.int32))
    return sc, B.SolveRegion(sc, abi.REGION_SUBDOMAIN, 0.0, sub, epsilon=1e-3)


def test_region_sampler_pdf_containment_moments():
    """RegionSampler (sampling.cpp:62-108) through generateSourceCache (cache.cpp:392-406):
    the reference's test_geometry.cpp:287-316 — unit square, 100000 unstratified samples,
    pdf = 1 and mean (0.5, 0.5) within 0.003 (plus E[x^2] = 1/3); a 256-gon disk, 2000
    stratified samples, pdf = 1/polygon area (FP32 storage) within 1e-3 of 1/pi, all inside."""
    pb = H.make_problem(H.kspec(), f=abi.make_field(abi.FIELD_CONSTANT, [1.0]))
    sc, region = _region_from_loop(O.rectangle_geometry([0, 0], [1, 1], [0, 0, 0, 0]))
    assert abs(region.area - 1.0) < 1e-14
    cfg = B.cache_config(nSource=100000, stratified=0)
    d = B.generate_source_cache(pb, region, cfg, 29, 0).download()
    assert len(d["pdf"]) == 100000
    np.testing.assert_allclose(d["pdf"], 1.0, rtol=1e-7)
    m = d["y"].mean(0)
    assert np.all(np.abs(m - 0.5) < 0.003), m
    m2 = (d["y"] ** 2).mean(0)
    assert np.all(np.abs(m2 - 1.0 / 3.0) < 0.003), m2
    assert np.all((d["y"] > 0) & (d["y"] < 1))
    disk = O.circle_geometry(segments=256)
    area = 0.5 * 256 * np.sin(2 * np.pi / 256)
    sc, region = _region_from_loop(disk)
    assert abs(region.area - area) < 1e-14 * area
    d = B.generate_source_cache(pb, region, B.cache_config(nSource=2000, stratified=1), 29, 1).download()
    np.testing.assert_allclose(d["pdf"], 1.0 / area, rtol=1e-7)
    assert np.all(np.abs(d["pdf"] - 1.0 / np.pi) < 1e-3)
    assert np.all(region.boundary.inside(d["y"]))
    assert np.all(O.RefScene(*disk).inside(d["y"]))


@pytest.mark.ref
@pytest.mark.parametrize("stratified", [0, 1])
def test_region_sampler_distribution_matches_reference(stratified):
    """The GPU source samples and the reference's RegionSampler on C3's Subdomain loop
    (a 5-star) draw from the same law: two-sample KS tests on x, y and the radius, and
    the means / second moments within 4 standard errors."""
    from scipy import stats

    c = configs.config3(scale=1 / 16)
    sc = B.Scene(c.vertices, c.segments, c.labels)
    sub = B.Scene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
    region = B.SolveRegion(sc, abi.REGION_SUBDOMAIN, c.region_offset, sub, epsilon=c.epsilon)
    rs = O.RefScene(c.vertices, c.segments, c.labels)
    rsub = O.RefScene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
    rr = O.RefRegion(rs, abi.REGION_SUBDOMAIN, c.region_offset, rsub, eps=c.epsilon)
    cfg = c.cache
    cfg.nSource, cfg.stratified = 65536, stratified
    g = B.generate_source_cache(c.problem, region, cfg, 5, 0).download()
    r = O.ref_generate_source_cache(c.problem, rr, cfg, 5, 0)
    assert len(g["y"]) == len(r["y"]) == 65536
    assert np.all(rsub.inside(g["y"]))
    np.testing.assert_allclose(g["pdf"], r["pdf"], rtol=1e-7)
    for name, a, b in (("x", g["y"][:, 0], r["y"][:, 0]), ("y", g["y"][:, 1], r["y"][:, 1]),
                       ("radius", np.hypot(*g["y"].T), np.hypot(*r["y"].T))):
        assert stats.ks_2samp(a, b).pvalue > 1e-3, name
    for k in range(2):
        for mom in (1, 2):
            a, b = g["y"][:, k] ** mom, r["y"][:, k] ** mom
            se = np.sqrt(a.var() / len(a) + b.var() / len(b))
            assert abs(a.mean() - b.mean()) < 4 * se, (k, mom)


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


def _near_band_points(v, s, l, n, rng):
    """points placed at distance l (1 + delta) from random segments' interiors, delta in
    {0, +-1e-15, +-1e-12, +-1e-9}: the band's edge, where an FP32 decision would flip"""
    ids = rng.integers(0, len(s), n)
    a, b = v[s[ids, 0]], v[s[ids, 1]]
    t = rng.uniform(0.05, 0.95, n)
    p = a + t[:, None] * (b - a)
    d = b - a
    nrm = np.stack([-d[:, 1], d[:, 0]], 1) / np.linalg.norm(d, axis=1)[:, None]  # left normal: inside of a CCW loop
    delta = rng.choice([0.0, 1e-15, -1e-15, 1e-12, -1e-12, 1e-9, -1e-9], n)
    return p + nrm * (l * (1.0 + delta))[:, None]


@pytest.mark.ref
@pytest.mark.parametrize("cid", [0, 1, 2, 3])
def test_mark_points_match_reference(cid):
    """markEvaluationPoints (cache.cpp:263-276) bit-exact: the fallback and gradientUnreliable
    flags equal the reference's on every point — disk points, the full C1/C2/C3 query grids,
    and points placed at the band's edge (distance l (1 +- 1e-15 ... 1e-9))."""
    rng = np.random.default_rng(2 + cid)
    if cid == 0:
        geom, pb, sc, region = _setup(H.disk_poisson)
        rs = O.RefScene(*geom)
        rr = O.RefRegion(rs, abi.REGION_WHOLE_DOMAIN, 0.05, eps=1e-3)
        cfg = B.cache_config(offset=0.05)
        r = np.sqrt(rng.uniform(0, 0.99, 4000))
        a = rng.uniform(0, 2 * np.pi, 4000)
        x = np.stack([r * np.cos(a), r * np.sin(a)], 1)
        v, s, lab = geom
        l = 0.05
    else:
        c = configs.CONFIGS[cid]()
        sc = B.Scene(c.vertices, c.segments, c.labels)
        rs = O.RefScene(c.vertices, c.segments, c.labels)
        cfg = c.cache
        if c.region_mode == abi.REGION_SUBDOMAIN:
            sub = B.Scene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
            region = B.SolveRegion(sc, abi.REGION_SUBDOMAIN, c.region_offset, sub, epsilon=c.epsilon)
            rsub = O.RefScene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
            rr = O.RefRegion(rs, abi.REGION_SUBDOMAIN, c.region_offset, rsub, eps=c.epsilon)
            x = c.points[rsub.inside(c.points)]
            v, s, lab = c.sub_vertices, c.sub_segments, None
        else:
            region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
            rr = O.RefRegion(rs, abi.REGION_WHOLE_DOMAIN, c.region_offset, eps=c.epsilon)
            x = c.points
            v, s, lab = c.vertices, c.segments, c.labels
        l = region.offset
    if lab is not None:
        s = s[lab == abi.DIRICHLET]
    x = np.concatenate([x, _near_band_points(v, s, l, 20000, rng)])
    pts = B.EvaluationPoints(x)
    B.mark_evaluation_points(sc, region, cfg, pts)
    st = pts.download()
    fb, gu = O.ref_mark_points(rs, rr, cfg, x)
    assert np.array_equal(st["fallback"], fb), int(np.sum(st["fallback"] != fb))
    assert np.array_equal(st["gradientUnreliable"], gu), int(np.sum(st["gradientUnreliable"] != gu))


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
