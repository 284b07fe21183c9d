"""The interior gather (splatSolution / splatGradient, cache.cpp:426-497) on the GPU
vs the double-precision oracle and the reference on IDENTICAL caches.

Bar (BASELINE.json north star): max_k |u_gpu - u_ref| / max(max|u_ref|, RMS(u_ref))
<= 1e-4 for u and for each gradient component. The caches are FP32-representable
(the GPU stores FP32), and the oracle consumes the same FP32-rounded values."""
import numpy as np
import pytest

import paper_2302_11825_b200 as B
from oracle import oracle as O
from paper_2302_11825_b200 import abi, configs
from tests import helpers as H

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _fp32(d):
    return {k: (np.asarray(v, np.float32).astype(np.float64) if np.asarray(v).dtype.kind == "f" else v)
            for k, v in d.items()}


def _gpu_splat(spec, cache, scache, x, value=True, gradient=True, fallback=None, voronoi=False):
    dim = spec.dim
    bc = B.BoundaryCache.from_arrays(cache["z"], cache["n"], cache["pdf"], cache["uHat"], cache["dHat"],
                                     cache.get("weight"), voronoi=voronoi) if cache is not None else None
    sc = B.SourceCache.from_arrays(scache["y"], scache["pdf"], scache["f"]) if scache is not None else None
    pts = B.EvaluationPoints(x, dim)
    if fallback is not None:
        pts.set_fallback(fallback)
    cfg = abi.SplatConfig(spec, 1e-12 * spec.scale, int(voronoi), 0)
    if value and gradient:
        B.splat_solution_gradient(bc, sc, pts, cfg)
    elif value:
        B.splat_solution(bc, sc, pts, cfg)
    else:
        B.splat_gradient(bc, sc, pts, cfg)
    return pts.download(), pts


@pytest.mark.parametrize("name", ["square_ux", "disk_poisson", "screened_disk"])
def test_gather_vs_reference_on_identical_cache(golden, name):
    g = golden("splat")
    k, sg, dim, scale = g[name + "_spec"]
    spec = H.kspec(int(k), sg, int(dim), scale)
    cache = _fp32({key: g[f"{name}_b_{key}"] for key in ("z", "n", "pdf", "uHat", "dHat", "weight")})
    scache = None
    if f"{name}_s_y" in g.files:
        scache = _fp32({key: g[f"{name}_s_{key}"] for key in ("y", "pdf", "f")})
    x = np.asarray(g[name + "_x"], np.float32).astype(np.float64)
    st, _ = _gpu_splat(spec, cache, scache, x)
    ref = O.oracle_splat(spec, 1e-12 * scale, cache, scache, x, value=True, gradient=True)
    for key in ("boundarySum", "sourceSum"):
        assert H.rel_err(st[key], ref[key]) <= TOL, key
    for key in ("boundaryGradSum", "sourceGradSum"):
        for c in range(2):
            assert H.rel_err(st[key][:, c], ref[key][:, c]) <= TOL, (key, c)
    # and the reference itself (non-rounded cache) agrees to FP32 input rounding
    assert H.rel_err(O.solution(st), O.solution(dict(
        boundarySum=g[name + "_boundarySum"], sourceSum=g[name + "_sourceSum"], nBoundary=g[name + "_nBoundary"],
        mSource=np.full(len(x), 0 if scache is None else len(scache["f"]))))) < 1e-3
    assert np.array_equal(st["nBoundary"], ref["nBoundary"]) and np.array_equal(st["mSource"], ref["mSource"])


def _config_cache(cfgfn, n_points=3000, seed=0, **kw):
    c = cfgfn(**kw)
    scene = B.Scene(c.vertices, c.segments, c.labels)
    if c.region_mode == abi.REGION_SUBDOMAIN:
        region = B.SolveRegion(scene, abi.REGION_SUBDOMAIN, c.region_offset, B.Scene(c.sub_vertices, c.sub_segments,
                                                                                        np.zeros(len(c.sub_segments))),
                               epsilon=c.epsilon)
    else:
        region = B.SolveRegion(scene, offset=c.region_offset, epsilon=c.epsilon)
    cache = B.generate_boundary_cache(scene, c.problem, region, c.cache, c.seed, 0)
    scache = B.generate_source_cache(c.problem, region, c.cache, c.seed, 0) if c.problem.f.kind else None
    rng = np.random.default_rng(seed)
    pts = c.points
    if c.region_mode == abi.REGION_SUBDOMAIN:
        pts = pts[region.boundary.inside(pts)]
    else:
        pts = pts[scene.inside(pts)]
    sel = pts[rng.choice(len(pts), size=min(n_points, len(pts)), replace=False)]
    return c, scene, region, cache, scache, sel


@pytest.mark.parametrize("which", [1, 2])
def test_gather_parity_baseline_configs_laplace(which):
    """C1 (u) and C2 (u, grad u) at full cache size, a point subset, vs the double oracle."""
    fn = configs.config1 if which == 1 else configs.config2
    c, scene, region, cache, _, x = _config_cache(fn, 2500)
    spec = H.kspec(0, 0.0, 2, scene.diagonal)
    cd = cache.download()
    st, _ = _gpu_splat(spec, cd, None, x, gradient=(which == 2))
    ref = O.oracle_splat(spec, 1e-12 * scene.diagonal, cd, None, np.asarray(x, np.float32).astype(float),
                         value=True, gradient=(which == 2))
    assert H.rel_err(O.solution(st), O.solution(ref)) <= TOL
    if which == 2:
        g, gr = O.gradient(st), O.gradient(ref)
        for c_ in range(2):
            assert H.rel_err(g[:, c_], gr[:, c_]) <= TOL


def test_gather_parity_config3_screened_with_source():
    """C3: screened sigma = 10 (K0/K1 in FP32), boundary + source samples, u and grad u."""
    c, scene, region, cache, scache, x = _config_cache(configs.config3, 600, scale=1 / 16, grid_n=256)
    spec = H.kspec(1, 10.0, 2, scene.diagonal)
    cd, sd = cache.download(), scache.download()
    st, _ = _gpu_splat(spec, cd, sd, x, gradient=True)
    ref = O.oracle_splat(spec, 1e-12 * scene.diagonal, cd, sd, np.asarray(x, np.float32).astype(float),
                         value=True, gradient=True)
    for key in ("boundarySum", "sourceSum"):
        assert H.rel_err(st[key], ref[key]) <= TOL, key
    for key in ("boundaryGradSum", "sourceGradSum"):
        for c_ in range(2):
            assert H.rel_err(st[key][:, c_], ref[key][:, c_]) <= TOL, (key, c_)


@pytest.mark.parametrize("kind,sigma", [(0, 0.0), (1, 1.0)])
def test_gather_parity_3d(kind, sigma):
    """3D Laplace / screened splats (the reference's 3D kernel templates, kernels.h:78-129)."""
    rng = np.random.default_rng(3)
    N, M, K = 3000, 700, 400
    zn = rng.normal(size=(N, 3))
    zn /= np.linalg.norm(zn, axis=1)[:, None]
    cache = _fp32(dict(z=zn, n=zn, pdf=np.full(N, 1 / (4 * np.pi)), uHat=rng.uniform(-1, 1, N),
                       dHat=rng.uniform(-1, 1, N), weight=np.zeros(N)))
    yy = rng.uniform(-0.5, 0.5, (M, 3))
    scache = _fp32(dict(y=yy, pdf=np.full(M, 1.0), f=rng.uniform(-2, 2, M)))
    x = np.asarray(rng.uniform(-0.6, 0.6, (K, 3)), np.float32).astype(float)
    spec = H.kspec(kind, sigma, 3, 2 * np.sqrt(3))
    st, _ = _gpu_splat(spec, cache, scache, x, gradient=True)
    ref = O.oracle_splat(spec, 1e-12 * spec.scale, cache, scache, x, value=True, gradient=True)
    for key in ("boundarySum", "sourceSum"):
        assert H.rel_err(st[key], ref[key]) <= TOL, key
    for key in ("boundaryGradSum", "sourceGradSum"):
        for c_ in range(3):
            assert H.rel_err(st[key][:, c_], ref[key][:, c_]) <= TOL, (key, c_)


def test_gather_bookkeeping():
    """test_cache.cpp:539-569 on the device: counts, coincident skip, fallback untouched, accumulation."""
    v, s, lab = O.rectangle_geometry([0, 0], [1, 1], [0, 0, 0, 0])
    osc = O.OracleScene(v, s, lab)
    z, n, pdf, _, _ = osc.boundary_sample(64, False, key=31)
    cache = _fp32(dict(z=z, n=n, pdf=pdf, uHat=z[:, 0], dHat=n[:, 0], weight=np.zeros(64)))
    y, ypdf = osc.region_sample(32, False, key=32)
    scache = _fp32(dict(y=y, pdf=ypdf, f=np.ones(32)))
    spec = H.kspec(0, 0, 2, osc.diagonal)
    bc = B.BoundaryCache.from_arrays(cache["z"], cache["n"], cache["pdf"], cache["uHat"], cache["dHat"])
    sc = B.SourceCache.from_arrays(scache["y"], scache["pdf"], scache["f"])
    cfg = abi.SplatConfig(spec, 1e-12 * osc.diagonal, 0, 0)
    pts = B.EvaluationPoints([[0.5, 0.5]])
    B.splat_solution(bc, sc, pts, cfg)
    st = pts.download()
    assert st["nBoundary"][0] == 64 and st["mSource"][0] == 32
    B.splat_solution(bc, sc, pts, cfg)
    st2 = pts.download()
    assert st2["nBoundary"][0] == 128 and st2["mSource"][0] == 64
    assert st2["boundarySum"][0] == 2 * st["boundarySum"][0]
    co = B.EvaluationPoints(cache["z"][:1])
    B.splat_solution(bc, sc, co, cfg)
    cst = co.download()
    assert cst["skipped"][0] == 1 and cst["nBoundary"][0] == 63 and np.isfinite(cst["boundarySum"][0])
    ref = O.oracle_splat(spec, 1e-12 * osc.diagonal, cache, scache, cache["z"][:1])
    assert H.rel_err(cst["boundarySum"], ref["boundarySum"]) <= TOL
    fb = B.EvaluationPoints([[0.5, 0.5], [0.3, 0.3]])
    fb.set_fallback([1, 0])
    B.splat_solution(bc, sc, fb, cfg)
    fst = fb.download()
    assert fst["nBoundary"][0] == 0 and fst["boundarySum"][0] == 0.0 and fst["nBoundary"][1] == 64


def test_gather_is_deterministic_and_shard_invariant():
    """Fixed summation order: bitwise repeatable, and splitting the points (multi-GPU
    sharding) gives bitwise the same sums (test_cache.cpp:321-347 analogue)."""
    c, scene, region, cache, _, x = _config_cache(configs.config2, 5000, scale=1 / 4)
    spec = abi.SplatConfig(H.kspec(0, 0, 2, scene.diagonal), 1e-12 * scene.diagonal, 0, 0)
    a = B.EvaluationPoints(x)
    B.splat_solution_gradient(cache, None, a, spec)
    b = B.EvaluationPoints(x)
    B.splat_solution_gradient(cache, None, b, spec)
    sa, sb = a.download(), b.download()
    assert np.array_equal(sa["boundarySum"], sb["boundarySum"])
    assert np.array_equal(sa["boundaryGradSum"], sb["boundaryGradSum"])
    sh = B.EvaluationPoints(x)
    half = len(x) // 3
    B.splat_range(cache, None, sh, spec, 0, half, True, True)
    B.splat_range(cache, None, sh, spec, half, len(x), True, True)
    ss = sh.download()
    assert np.array_equal(ss["boundarySum"], sa["boundarySum"])
    assert np.array_equal(ss["boundaryGradSum"], sa["boundaryGradSum"])
    assert np.array_equal(ss["nBoundary"], sa["nBoundary"])


def test_exact_data_winding_number():
    """test_cache.cpp:392-412: u == 1 data, the double layer gives 1 inside and 0 outside."""
    v, s, lab = O.circle_geometry(segments=256)
    osc = O.OracleScene(v, s, lab)
    spec = abi.SplatConfig(H.kspec(0, 0, 2, osc.diagonal), 1e-12 * osc.diagonal, 0, 0)
    ins, outs = [], []
    for seed in range(150):
        z, n, pdf, _, _ = osc.boundary_sample(128, False, key=O.oracle_lib().or_mixkey(1, seed))
        bc = B.BoundaryCache.from_arrays(z, n, pdf, np.ones(128), np.zeros(128))
        pts = B.EvaluationPoints([[0.3, 0.4], [2.0, 0.0]])
        B.splat_solution(bc, None, pts, spec)
        u = pts.solution()
        ins.append(u[0])
        outs.append(u[1])
    ins, outs = np.array(ins), np.array(outs)
    assert abs(ins.mean() - 1.0) <= 3 * ins.std(ddof=1) / np.sqrt(len(ins))
    assert abs(outs.mean()) <= 4 * outs.std(ddof=1) / np.sqrt(len(outs))


def test_voronoi_weights_gather():
    rng = np.random.default_rng(9)
    N = 512
    th = np.sort(rng.uniform(0, 2 * np.pi, N))
    z = np.stack([np.cos(th), np.sin(th)], 1)
    w = np.diff(np.concatenate([th[-1:] - 2 * np.pi, th, th[:1] + 2 * np.pi]))
    w = 0.5 * (w[:-1] + w[1:])
    cache = _fp32(dict(z=z, n=z, pdf=np.full(N, 1 / (2 * np.pi)), uHat=z[:, 0], dHat=z[:, 0], weight=w))
    x = np.asarray(rng.uniform(-0.5, 0.5, (200, 2)), np.float32).astype(float)
    spec = H.kspec(0, 0, 2, 2 * np.sqrt(2))
    st, _ = _gpu_splat(spec, cache, None, x, gradient=False, voronoi=True)
    ref = O.oracle_splat(spec, 1e-12 * spec.scale, cache, None, x, voronoi=True)
    assert H.rel_err(st["boundarySum"], ref["boundarySum"]) <= TOL


@pytest.mark.parametrize("name", ["square_ux", "disk_poisson"])
def test_fp64_gather_matches_reference_to_rounding(golden, name):
    """The FP64 variant (BASELINE C1 "u (fp32 and fp64)"): on the FP32-stored cache the
    reference's own double loop and the GPU's FP64 loop agree to ~1e-13."""
    g = golden("splat")
    k, sg, dim, scale = g[name + "_spec"]
    spec = H.kspec(int(k), sg, int(dim), scale)
    cache = _fp32({key: g[f"{name}_b_{key}"] for key in ("z", "n", "pdf", "uHat", "dHat", "weight")})
    scache = None
    if f"{name}_s_y" in g.files:
        scache = _fp32({key: g[f"{name}_s_{key}"] for key in ("y", "pdf", "f")})
    x = np.asarray(g[name + "_x"], np.float64)
    bc = B.BoundaryCache.from_arrays(cache["z"], cache["n"], cache["pdf"], cache["uHat"], cache["dHat"])
    sc = B.SourceCache.from_arrays(scache["y"], scache["pdf"], scache["f"]) if scache is not None else None
    pts = B.EvaluationPoints(x)
    cfg = abi.SplatConfig(spec, 1e-12 * scale, 0, 0, 1)
    B.splat_solution_gradient(bc, sc, pts, cfg)
    st = pts.download()
    ref = O.oracle_splat(spec, 1e-12 * scale, cache, scache, x, value=True, gradient=True)
    for key in ("boundarySum", "sourceSum"):
        assert H.rel_err(st[key], ref[key]) <= 1e-12, (key, H.rel_err(st[key], ref[key]))
    for key in ("boundaryGradSum", "sourceGradSum"):
        for c in range(2):
            assert H.rel_err(st[key][:, c], ref[key][:, c]) <= 1e-12, (key, c)
    assert np.array_equal(st["nBoundary"], ref["nBoundary"]) and np.array_equal(st["skipped"], ref["skipped"])
    # the exact per-pair coincidence test: a point on a sample skips exactly that sample
    on = B.EvaluationPoints(cache["z"][:3])
    B.splat_solution(bc, sc, on, cfg)
    so = on.download()
    ro = O.oracle_splat(spec, 1e-12 * scale, cache, scache, cache["z"][:3])
    assert np.array_equal(so["skipped"], ro["skipped"]) and np.all(so["skipped"] >= 1)
    assert H.rel_err(so["boundarySum"], ro["boundarySum"]) <= 1e-12


def test_fp64_gather_3d_and_c1_config():
    rng = np.random.default_rng(5)
    z = rng.normal(size=(3000, 3))
    z /= np.linalg.norm(z, axis=1)[:, None]
    cache = dict(z=z, n=z, pdf=np.full(3000, 1 / (4 * np.pi)), uHat=rng.uniform(-1, 1, 3000),
                 dHat=rng.uniform(-1, 1, 3000), weight=np.zeros(3000))
    cache = _fp32(cache)
    x = rng.uniform(-0.5, 0.5, (700, 3))
    spec = H.kspec(0, 0, 3, 2.0)
    bc = B.BoundaryCache.from_arrays(cache["z"], cache["n"], cache["pdf"], cache["uHat"], cache["dHat"])
    pts = B.EvaluationPoints(x, 3)
    B.splat_solution_gradient(bc, None, pts, abi.SplatConfig(spec, 2e-12, 0, 0, 1))
    st = pts.download()
    ref = O.oracle_splat(spec, 2e-12, cache, None, x, value=True, gradient=True)
    assert H.rel_err(st["boundarySum"], ref["boundarySum"]) <= 1e-12
    for c in range(3):
        assert H.rel_err(st["boundaryGradSum"][:, c], ref["boundaryGradSum"][:, c]) <= 1e-12
    # C1's cache through both precisions: the FP32 gather sits within its 1e-4 bar of FP64
    c, scene, region, cache1, _, x1 = _config_cache(configs.config1, 4000)
    spec1 = H.kspec(0, 0, 2, scene.diagonal)
    a, b = B.EvaluationPoints(x1), B.EvaluationPoints(x1)
    B.splat_solution(cache1, None, a, abi.SplatConfig(spec1, 1e-12 * scene.diagonal, 0, 0, 0))
    B.splat_solution(cache1, None, b, abi.SplatConfig(spec1, 1e-12 * scene.diagonal, 0, 0, 1))
    assert H.rel_err(a.solution(), b.solution()) <= TOL
    with pytest.raises(B.InvalidArgument):
        B.splat_solution(cache1, None, a, abi.SplatConfig(H.kspec(1, 1.0, 2, 2.0), 1e-12, 0, 0, 1))
