"""Gather parity at the configs' real scale (SURVEY §8d bar, per point:
max_k |u_gpu - u_ref| / max(|u_ref,k|, RMS(u_ref)) <= 1e-4, also per gradient
component): the caches are the GPU's own full-size caches of C3 (65,536 boundary +
65,536 source samples, screened sigma = 10), C4 (262,144 samples) and C5 (1,048,576
samples on the soup's shell, screened sigma = 1). The query points include points
within one sample spacing of the boundary, where the near-singular FP32 terms are
largest. The reference side is the reference's own splatSolution / splatGradient
(2D, oracle/_ref, threaded) or splatSolution's loop over its 3D kernel templates
(ref_splat3), in double, on the identical FP32 cache."""
import numpy as np
import pytest

import paper_2302_11825_b200 as B
from oracle import oracle as O
from paper_2302_11825_b200 import abi, configs
from tests import helpers as H

pytestmark = [pytest.mark.gpu, pytest.mark.ref]
TOL = 1e-4


def _points_near(cache, spacing, k, rng, inward):
    """k points at distance U(0.1, 1) x spacing from random cache samples, on the interior side"""
    i = rng.choice(len(cache["pdf"]), k, replace=False)
    d = rng.uniform(0.1, 1.0, k) * spacing
    return cache["z"][i] + inward * d[:, None] * cache["n"][i]


def test_gather_parity_config3_full_cache():
    c = configs.config3()
    sc = B.Scene(c.vertices, c.segments, c.labels)
    sub = B.Scene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
    region = B.SolveRegion(sc, abi.REGION_SUBDOMAIN, c.region_offset, sub, epsilon=c.epsilon)
    cache = B.generate_boundary_cache(sc, c.problem, region, c.cache, c.seed, 0)
    scache = B.generate_source_cache(c.problem, region, c.cache, c.seed, 0)
    cd, sd = cache.download(), scache.download()
    assert len(cd["pdf"]) == 65536 and len(sd["pdf"]) == 65536
    rng = np.random.default_rng(7)
    pts = c.points[region.boundary.inside(c.points)]
    length = float(np.sum(np.linalg.norm(np.diff(np.vstack([c.sub_vertices, c.sub_vertices[:1]]), axis=0), axis=1)))
    near = _points_near(cd, length / 65536, 48, rng, -1.0)  # the region loop is CCW: inside is -n
    near = near[region.boundary.inside(near)]
    x = np.vstack([pts[rng.choice(len(pts), 80, replace=False)], near])
    x = np.asarray(x, np.float32).astype(np.float64)
    p = B.EvaluationPoints(x)
    spec = B.make_splat_config(sc, c.problem, c.cache)
    B.splat_solution_gradient(cache, scache, p, spec)
    st = p.download()
    ks = H.kspec(1, 10.0, 2, sc.diagonal)
    ref = O.ref_splat(ks, 1e-12 * sc.diagonal, cd, sd, x, value=True, gradient=True, threads=0)
    assert H.rel_err_pointwise(O.solution(st), O.solution(ref)) <= TOL
    g, gr = O.gradient(st), O.gradient(ref)
    for k in range(2):
        assert H.rel_err_pointwise(g[:, k], gr[:, k]) <= TOL, k
    assert np.array_equal(st["nBoundary"], ref["nBoundary"]) and np.array_equal(st["mSource"], ref["mSource"])


def _build3(cid):
    c = configs.CONFIGS[cid]()
    if "components" in c.extra:
        tris, labels = configs.soup_shell(c)
        comps = configs.soup_components(c)
        c.segments, c.labels = tris, labels
        sc = B.Scene.mesh3(c.vertices, c.segments, c.labels)

        def inside(x):
            keep = np.zeros(len(x), bool)
            for m in comps:
                keep |= m.inside(x)
            return keep
    else:
        sc = B.Scene.mesh3(c.vertices, c.segments, c.labels)
        inside = sc.inside
    region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
    return c, sc, region, inside


@pytest.mark.parametrize("cid", [4, 5])
def test_gather_parity_3d_full_cache(cid):
    c, sc, region, inside = _build3(cid)
    cache = B.generate_boundary_cache(sc, c.problem, region, c.cache, c.seed, 0)
    cd = cache.download()
    N = len(cd["pdf"])
    assert N == c.cache.nBoundary
    rng = np.random.default_rng(11)
    V, F = c.vertices, c.segments
    area = 0.5 * np.linalg.norm(np.cross(V[F[:, 1]] - V[F[:, 0]], V[F[:, 2]] - V[F[:, 0]]), axis=1).sum()
    spacing = np.sqrt(area / N)
    near = _points_near(cd, spacing, 400, rng, -1.0)  # outward normals: inside is -n
    near = near[inside(near)][:128]
    far = c.points[:4096]
    far = far[inside(far)][:128]
    x = np.asarray(np.vstack([far, near]), np.float32).astype(np.float64)
    assert len(near) >= 64
    p = B.EvaluationPoints(x, 3)
    spec = B.make_splat_config(sc, c.problem, c.cache)
    B.splat_solution(cache, None, p, spec)
    st = p.download()
    ks = H.kspec(c.problem.kernel.kind, c.problem.kernel.sigma, 3, sc.diagonal)
    ref = O.ref_splat3(ks, 1e-12 * sc.diagonal, cd, x, threads=0)
    u, ur = st["boundarySum"] / st["nBoundary"], ref["boundarySum"] / ref["nBoundary"]
    assert np.array_equal(st["nBoundary"], ref["nBoundary"])
    assert H.rel_err_pointwise(u, ur) <= TOL, H.rel_err_pointwise(u, ur)
