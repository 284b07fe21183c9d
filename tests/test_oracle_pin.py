"""Pins the C restatement (oracle/bvc_oracle.c) before anything is checked against it.

Two anchors: (a) golden vectors produced by the reference itself (tests/golden/,
made by tests/golden/make_golden.py from oracle/_ref), and (b) known answers the
reference's own tests hold (test_kernels.cpp:43-108, 311-329; test_cache.cpp:392-569).
Runs on CPU only.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_2302_11825_b200 import abi
from tests import helpers as H


def test_rng_matches_reference_bitwise(golden):
    g = golden("rng")
    L = O.oracle_lib()
    for (seed, stream), ref in zip(g["cases"], g["uniforms"]):
        out = np.zeros(16)
        L.or_rng_uniforms(int(seed), int(stream), 16, out)
        assert np.array_equal(out, ref)
    for (a, b), ref in zip([(0, 0), (0x1002, 3), (123456789, 42)], g["mixkey"]):
        assert L.or_mixkey(a, b) == int(ref)


def test_bessel_known_answers_and_reference(golden):
    L = O.oracle_lib()
    # frozen values of test_kernels.cpp:313-318
    assert L.or_bessel_k0(1.0) == pytest.approx(0.42102443824070834, rel=1e-12)
    assert L.or_bessel_k1(1.0) == pytest.approx(0.6019072301972346, rel=1e-12)
    assert L.or_bessel_k0(800.0) == 0.0 and L.or_bessel_i0(0.0) == 1.0
    g = golden("bessel")
    fns = [L.or_bessel_k0, L.or_bessel_k1, L.or_bessel_i0, L.or_bessel_i1]
    for w, f in enumerate(fns):
        got = np.array([f(t) for t in g["t"]])
        np.testing.assert_allclose(got, g["values"][w], rtol=1e-12, atol=0)
    # dK0/dt = -K1 (test_kernels.cpp:321-325)
    for t in (0.5, 1.0, 2.0):
        d = 1e-6 * t
        fd = (L.or_bessel_k0(t + d) - L.or_bessel_k0(t - d)) / (2 * d)
        assert fd == pytest.approx(-L.or_bessel_k1(t), rel=1e-7)


@pytest.mark.parametrize("name", ["p2", "s2", "p3", "s3", "s2big"])
def test_kernel_formulas_match_reference(golden, name):
    g = golden("kernels")
    k, sg, dim, sc = g[name + "_spec"]
    spec = H.kspec(int(k), sg, int(dim), sc)
    x, y, n, ref = g[name + "_x"], g[name + "_y"], g[name + "_n"], g[name + "_out"]
    out = np.zeros_like(ref)
    assert O.oracle_lib().or_eval_kernels(C.byref(spec), x.ravel(), y.ravel(), n.ravel(), len(x), out.ravel()) == 0
    np.testing.assert_allclose(out, ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())


def test_kernel_reference_values():
    """test_kernels.cpp:43-108: signs and magnitudes of the reference convention."""
    L = O.oracle_lib()

    def ev(spec, x, y, n):
        d = spec.dim
        out = np.zeros(2 + 2 * d)
        assert L.or_eval_kernels(C.byref(spec), np.array(x, float), np.array(y, float), np.array(n, float), 1, out) == 0
        return out

    p2 = ev(H.kspec(), [0, 0], [1, 0], [1, 0])
    assert p2[0] == pytest.approx(0.0, abs=1e-15)                    # ln(1)/2pi
    assert p2[1] == pytest.approx(-1 / (2 * np.pi), rel=1e-14)       # dG/dx
    assert p2[3] == pytest.approx(1 / (2 * np.pi), rel=1e-14)        # Poisson kernel
    assert p2[4] == pytest.approx(1 / (2 * np.pi), rel=1e-14)
    g3 = ev(H.kspec(0, 0, 3), [0, 0, 0], [0.5, 0, 0], [1, 0, 0])
    assert g3[0] < 0 and abs(g3[0]) == pytest.approx(1 / (2 * np.pi), rel=1e-14)
    s3 = ev(H.kspec(1, 1.0, 3), [0, 0, 0], [1, 0, 0], [1, 0, 0])
    assert s3[0] == pytest.approx(-np.exp(-1) / (4 * np.pi), rel=1e-14)


def test_geometry_brute_force_matches_reference_bvh(golden):
    g = golden("geometry")
    for k in range(3):
        sc = O.OracleScene(g[f"s{k}_v"], g[f"s{k}_s"], g[f"s{k}_lab"])
        q, d = g[f"s{k}_q"], g[f"s{k}_d"]
        for filt in (abi.FILTER_ANY, abi.FILTER_DIRICHLET, abi.FILTER_NEUMANN):
            p, dist, seg, _ = sc.closest_point(q, filt)
            np.testing.assert_allclose(dist, g[f"s{k}_cp{filt}_dist"], rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(sc.silhouette_distance(q), g[f"s{k}_sil"], rtol=1e-14)
        for filt in (abi.FILTER_ANY, abi.FILTER_NEUMANN):
            t, seg, _, _ = sc.intersect_ray(q, d, np.inf, filt, 0.0)
            np.testing.assert_allclose(t, g[f"s{k}_ray{filt}_t"], rtol=1e-13)
            assert np.array_equal(seg, g[f"s{k}_ray{filt}_seg"])
        assert np.array_equal(sc.inside(q), g[f"s{k}_inside"])


def test_samplers_match_reference(golden):
    g = golden("sampler")
    sc = O.OracleScene(g["v"], g["s"], g["lab"])
    p, n, pdf, seg, arc = sc.boundary_sample(128, True, key=777)
    np.testing.assert_allclose(p, g["strat_p"], rtol=0, atol=1e-15)
    assert np.array_equal(seg, g["strat_seg"])
    np.testing.assert_allclose(arc, g["strat_arc"], rtol=1e-14)
    p2, *_ = sc.boundary_sample(128, False, key=778)
    np.testing.assert_allclose(p2, g["plain_p"], atol=1e-15)
    rp, rpdf = sc.region_sample(200, True, key=779)
    np.testing.assert_allclose(rp, g["region_strat"], atol=1e-15)
    rp2, _ = sc.region_sample(200, False, key=780)
    np.testing.assert_allclose(rp2, g["region_plain"], atol=1e-15)
    np.testing.assert_allclose(rpdf, g["region_pdf"], rtol=1e-14)


def _walk_problems():
    return {"disk_linear": (H.disk_linear(), 0), "disk_poisson": (H.disk_poisson(), 0),
            "mixed": (H.square_mixed(), 1), "vertical": (H.vertical(), 1), "screened": (H.screened_constant(), 0)}


@pytest.mark.parametrize("name", ["disk_linear", "disk_poisson", "mixed", "vertical", "screened"])
def test_walks_reproduce_reference_streams(golden, name):
    """Same xoshiro streams => the restated walks equal the reference's (pointwise.cpp:125-186)."""
    g = golden("walks")
    ((v, s, lab), pb), kind = _walk_problems()[name]
    sc = O.OracleScene(v, s, lab)
    cfg = abi.default_walk_config()
    cfg.nWalks, cfg.seed = 20000, {"disk_linear": 2, "disk_poisson": 3, "mixed": 6, "vertical": 7, "screened": 4}[name]
    out = sc.solve(pb, g[name + "_x"], cfg, kind)
    ref = g[name]
    assert out[0] == pytest.approx(ref[0], rel=1e-9, abs=1e-12)
    assert out[1] == pytest.approx(ref[1], rel=1e-9)
    assert out[2] == ref[2] and out[3] == ref[3]


def test_gradient_estimators_reproduce_reference(golden):
    g = golden("walks")
    (v, s, lab), pb = H.disk_poisson()
    sc = O.OracleScene(v, s, lab)
    cfg = abi.default_walk_config()
    cfg.nWalks, cfg.seed = 20000, 12
    out = sc.gradient(pb, g["grad_disk_poisson_x"], cfg)
    np.testing.assert_allclose(out[:4], g["grad_disk_poisson"][:4], rtol=1e-9)
    cfg.seed = 13
    out = sc.gradient(pb, g["dn_disk_poisson_x"], cfg, normal=[1.0, 0.0])
    np.testing.assert_allclose(out[:2], g["dn_disk_poisson"][:2], rtol=1e-9)
    (v, s, lab), pb = H.screened_constant()
    sc = O.OracleScene(v, s, lab)
    cfg.seed = 14
    out = sc.gradient(pb, g["grad_screened_x"], cfg)
    np.testing.assert_allclose(out[:4], g["grad_screened"][:4], rtol=1e-8, atol=1e-12)


@pytest.mark.parametrize("name", ["square_ux", "disk_poisson", "screened_disk"])
def test_splat_restatement_matches_reference(golden, name):
    g = golden("splat")
    k, sg, dim, sc = g[name + "_spec"]
    spec = H.kspec(int(k), sg, int(dim), sc)
    cache = {key: g[f"{name}_b_{key}"] for key in ("z", "n", "pdf", "uHat", "dHat", "weight")}
    scache = None
    if f"{name}_s_y" in g.files:
        scache = {key: g[f"{name}_s_{key}"] for key in ("y", "pdf", "f")}
    st = O.oracle_splat(spec, 1e-12 * sc, cache, scache, g[name + "_x"], value=True, gradient=True)
    for key in ("boundarySum", "sourceSum", "boundaryGradSum", "sourceGradSum"):
        np.testing.assert_allclose(st[key], g[f"{name}_{key}"], rtol=1e-11, atol=1e-12)
    assert np.array_equal(st["nBoundary"], g[name + "_nBoundary"])
    assert np.array_equal(st["skipped"], g[name + "_skipped"])


def test_splat_bookkeeping():
    """test_cache.cpp:539-569: counts accumulate, a coincident sample is skipped, fallback untouched."""
    v, s, lab = O.rectangle_geometry([0, 0], [1, 1], [0, 0, 0, 0])
    sc = O.OracleScene(v, s, lab)
    z, n, pdf, seg, arc = sc.boundary_sample(64, False, key=31)
    cache = dict(z=z, n=n, pdf=pdf, uHat=z[:, 0], dHat=n[:, 0], weight=np.zeros(64))
    y, ypdf = sc.region_sample(32, False, key=32)
    scache = dict(y=y, pdf=ypdf, f=np.ones(32))
    spec = H.kspec(0, 0, 2, sc.diagonal)
    st = O.oracle_splat(spec, 1e-12 * sc.diagonal, cache, scache, [[0.5, 0.5]])
    assert st["nBoundary"][0] == 64 and st["mSource"][0] == 32
    st = O.oracle_splat(spec, 1e-12 * sc.diagonal, cache, scache, [[0.5, 0.5]], state=st)
    assert st["nBoundary"][0] == 128 and st["mSource"][0] == 64
    co = O.oracle_splat(spec, 1e-12 * sc.diagonal, cache, scache, z[:1])
    assert co["skipped"][0] == 1 and co["nBoundary"][0] == 63
    fb = O.oracle_splat(spec, 1e-12 * sc.diagonal, cache, scache, [[0.5, 0.5]], fallback=[1])
    assert fb["nBoundary"][0] == 0


@pytest.mark.ref
def test_generate_boundary_cache_restatement_matches_reference(golden):
    """generateBoundaryCache restated (cache.cpp:301-390) on the reference's region."""
    g = golden("cache")
    (v, s, lab), pb = H.square_mixed()
    rs = O.RefScene(v, s, lab)
    rg = O.RefRegion(rs, abi.REGION_WHOLE_DOMAIN, 0.05, eps=1e-3)
    sc = O.OracleScene(v, s, lab)
    region = O.OracleScene(rg.vertices, rg.segments, rg.labels)
    cfg = abi.default_cache_config()
    cfg.nBoundary, cfg.nWalksNeumann, cfg.nWalksDirichlet, cfg.offset = 48, 8, 16, 0.05
    cfg.walk.epsilon = 1e-3
    N = 48
    z, n, pdf, u, d, arc = (np.zeros((N, 2)), np.zeros((N, 2)), np.zeros(N), np.zeros(N), np.zeros(N), np.zeros(N))
    seg = np.zeros(N, np.int32)
    stats = np.zeros(4, np.int64)
    e = O.oracle_lib().or_generate_boundary_cache(sc.h, C.byref(pb), region.h, rg.kinds.astype(np.int32),
                                                   rg.source.astype(np.int32), C.byref(cfg), 11, 0, 0, N,
                                                   z.ravel(), n.ravel(), pdf, u, d, seg, arc, stats)
    assert e == 0
    np.testing.assert_allclose(z, g["z"], atol=1e-15)
    np.testing.assert_allclose(u, g["uHat"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(d, g["dHat"], rtol=1e-9, atol=1e-9)
    assert stats[1] == g["stats"][1]


def _clamp_fixture(g):
    cache = {key: g[f"b_{key}"] for key in ("z", "n", "pdf", "uHat", "dHat", "weight")}
    scache = {key: g[f"s_{key}"] for key in ("y", "pdf", "f")}
    return cache, scache


def test_clamped_splat_restatement_matches_reference(golden):
    """correctedBoundarySplat (ClampOnly) / ball-kernel greensValue / correctedSourceSplat
    loops (cache.cpp:410-416, 512-524, 573-582) vs the reference on identical caches."""
    g = golden("clamp")
    cache, scache = _clamp_fixture(g)
    diag = 2.0 * np.sqrt(2.0)  # bounding-box diagonal of the unit 256-gon
    spec = H.kspec(0, 0, 2, diag)
    for i, (mode, c) in enumerate(g["cases"]):
        st = O.oracle_clamped_splat(spec, 1e-12 * diag, cache, scache, g["x"], int(mode), float(c), g["ballRadius"])
        for key in ("boundarySum", "sourceSum"):
            np.testing.assert_allclose(st[key], g[f"{i}_{key}"], rtol=1e-12, atol=1e-14)
        for key in ("nBoundary", "mSource", "skipped"):
            assert np.array_equal(st[key], g[f"{i}_{key}"])
    # an infinite bound is the plain splat (test_cache.cpp:748-764)
    inf = O.oracle_clamped_splat(spec, 1e-12 * diag, cache, None, g["x"], 1, np.inf)
    plain = O.oracle_splat(spec, 1e-12 * diag, cache, None, g["x"])
    assert np.array_equal(inf["boundarySum"], plain["boundarySum"])


def test_ball_radius_is_farthest_region_vertex(golden):
    """markEvaluationPoints' ballRadius (cache.cpp:268-274)."""
    g = golden("clamp")
    x, v = g["x"], g["region_v"]
    R = np.max(np.linalg.norm(v[None, :, :] - x[:, None, :], axis=2), axis=1)
    np.testing.assert_allclose(R, g["ballRadius"], rtol=1e-15)
