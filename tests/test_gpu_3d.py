"""3D triangle-mesh path (BASELINE configs 4-5). The reference has no 3D walks
(pointwise.cpp:23), so walk parity is against closed forms: on a sphere with
harmonic Dirichlet data u = g; the 3D gather is pinned against the restated loop
in test_gpu_gather.py::test_gather_parity_3d."""
import numpy as np
import pytest

import paper_2302_11825_b200 as B
from paper_2302_11825_b200 import abi, configs

pytestmark = pytest.mark.gpu

HARMONIC = abi.make_field(abi.FIELD_QUADRATIC3, [0.1, 0.3, -0.2, 0.5, -0.5, -0.5, 1.0, 1.0, 0.0, 0.0])


def g_exact(x):
    return 0.1 + 0.3 * x[:, 0] - 0.2 * x[:, 1] + 0.5 * x[:, 2] - 0.5 * x[:, 0] ** 2 - 0.5 * x[:, 1] ** 2 + \
        x[:, 2] ** 2 + x[:, 0] * x[:, 1]


def grad_exact(x):
    return np.stack([0.3 - x[:, 0] + x[:, 1], -0.2 - x[:, 1] + x[:, 0], 0.5 + 2 * x[:, 2]], 1)


@pytest.fixture(scope="module")
def sphere():
    V, F = configs.icosphere(4)
    return V, F, B.Scene.mesh3(V, F, np.zeros(len(F), np.int32))


def test_mesh_queries(sphere):
    V, F, sc = sphere
    rng = np.random.default_rng(1)
    x = rng.normal(size=(2000, 3))
    x *= (rng.uniform(0.0, 1.3, 2000) / np.linalg.norm(x, axis=1))[:, None]
    p, d, tri, _ = sc.closest_point(x)
    # brute force over all triangles (vertex/edge/face distance via dense sampling is too coarse; use the
    # support-plane distance as a lower bound and the returned point's distance as exact)
    r = np.linalg.norm(x, axis=1)
    inner = np.min(np.linalg.norm(V, axis=1))
    assert np.all(tri >= 0)
    assert np.all(np.abs(np.linalg.norm(p - x, axis=1) - d) < 1e-5)
    assert np.all(d <= np.abs(r - 1.0) + 0.02)  # the polyhedron is within 1 - inner of the sphere
    ins = sc.inside(x)
    assert np.all(ins[r < inner - 1e-3]) and not np.any(ins[r > 1.0 + 1e-3])


def test_cache_3d_closed_form(sphere):
    V, F, sc = sphere
    pb = B.problem(B.poisson(3), g=HARMONIC)
    region = B.SolveRegion(sc, offset=0.05, epsilon=1e-3)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3), nBoundary=512, nWalksNeumann=256, nWalksDirichlet=1024,
                         offset=0.05)
    st = {}
    c = B.generate_boundary_cache(sc, pb, region, cfg, 3, 0, stats=st).download()
    assert c["z"].shape == (512, 3) and st["cacheWalks"] == 512 * (256 + 1024)
    du = c["uHat"] - g_exact(c["z"])
    dd = c["dHat"] - np.sum(c["n"] * grad_exact(c["z"]), 1)
    assert abs(du.mean()) <= 4 * du.std(ddof=1) / np.sqrt(len(du)) + 2e-3   # O(eps) shell bias allowance
    assert abs(dd.mean()) <= 4 * dd.std(ddof=1) / np.sqrt(len(dd))
    assert du.std() < 0.05


def test_update_solution_3d_matches_harmonic_data(sphere):
    V, F, sc = sphere
    pb = B.problem(B.poisson(3), g=HARMONIC)
    region = B.SolveRegion(sc, offset=0.02, epsilon=1e-3)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3, nWalks=256), nBoundary=8192, nWalksNeumann=64,
                         nWalksDirichlet=256, offset=0.02)
    rng = np.random.default_rng(2)
    x = rng.normal(size=(4000, 3))
    x *= (0.99 * rng.uniform(0, 1, 4000) ** (1 / 3) / np.linalg.norm(x, axis=1))[:, None]
    x = x[sc.inside(x)]
    pts = B.EvaluationPoints(x, 3)
    B.mark_evaluation_points(sc, region, cfg, pts)
    for r in range(4):
        B.update_solution(sc, pb, region, cfg, pts, 9, r, gradients=True)
    st = pts.download()
    u = pts.solution(st)
    fb = st["fallback"]
    assert fb.sum() > 0 and np.all(st["walkCount"][fb] == 4 * 256), (fb.sum(), st["walkCount"][fb][:5])
    err = u - g_exact(x)
    assert np.all(np.isfinite(u))
    # away from the region boundary (the splat estimate is heavy-tailed within a sample
    # spacing of the cache surface, as in 2D)
    deep = np.linalg.norm(x, axis=1) < 0.9
    rms_in, rms_fb = np.sqrt(np.mean(err[deep] ** 2)), np.sqrt(np.mean(err[fb] ** 2))
    assert rms_in < 0.05 and rms_fb < 0.05, (rms_in, rms_fb)
    # unbiasedness: all points of one round share one cache, so their errors are one
    # correlated field; independent rounds are the unit of replication
    means = []
    for r in range(8):
        p = B.EvaluationPoints(x[deep], 3)
        B.mark_evaluation_points(sc, region, cfg, p)
        B.update_solution(sc, pb, region, cfg, p, 100 + r, 0)
        means.append(np.mean(p.solution() - g_exact(x[deep])))
    means = np.array(means)
    assert abs(means.mean()) <= 4 * means.std(ddof=1) / np.sqrt(len(means)) + 2e-3, means
    u2, g2 = pts.read_solution(gradient=True)
    assert np.allclose(u2, u, rtol=1e-12, atol=1e-12) and g2.shape == (len(x), 3)


def test_screened_mixed_3d_runs_and_is_bounded():
    """C5-style physics on one sphere: screened sigma = 1, Neumann cap (n.z > 0.5) with h = 0,
    Dirichlet g = 1 elsewhere: 0 < u <= 1 (maximum principle) and deterministic per seed."""
    V, F = configs.icosphere(4)
    n = np.cross(V[F[:, 1]] - V[F[:, 0]], V[F[:, 2]] - V[F[:, 0]])
    lab = (n[:, 2] / np.linalg.norm(n, axis=1) > 0.5).astype(np.int32)
    sc = B.Scene.mesh3(V, F, lab)
    pb = B.problem(B.screened(1.0, 3), g=abi.make_field(abi.FIELD_CONSTANT, [1.0]))
    region = B.SolveRegion(sc, offset=0.02, epsilon=1e-3)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3, nWalks=64), nBoundary=1024, nWalksNeumann=64,
                         nWalksDirichlet=64, offset=0.02)
    st = {}
    c = B.generate_boundary_cache(sc, pb, region, cfg, 5, 0, stats=st).download()
    kinds = region.kinds[c["segment"]]
    assert np.all(c["dHat"][kinds == abi.SEG_KNOWN_NEUMANN] == 0.0)
    assert np.all((c["uHat"] > 0) & (c["uHat"] <= 1.0 + 1e-6))
    c2 = B.generate_boundary_cache(sc, pb, region, cfg, 5, 0).download()
    assert np.array_equal(c["uHat"], c2["uHat"])
    assert st["cacheTruncated"] <= 1e-4 * st["cacheWalks"]


def test_c5_bvc_agrees_with_pointwise_walks():
    """C5 has no reference path and no closed form: its self-consistency check.
    On C5's own soup (shell of the 8 displaced spheres, sigma = 1, Neumann caps), the BVC
    estimate at interior points (mean over independent rounds) agrees with the pointwise
    WoSt estimate (wostSolve, pointwise.h:66) at the same points: |z| < 3 up to an O(eps)
    shell allowance, for all but a binomial allowance of the points."""
    c = configs.config5(scale=1 / 32, n_points=1000)
    tris, labels = configs.soup_shell(c)
    comps = configs.soup_components(c)
    sc = B.Scene.mesh3(c.vertices, tris, labels)
    region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
    rng = np.random.default_rng(11)
    cand = c.points[rng.permutation(len(c.points))[:4000]]
    inside = np.zeros(len(cand), bool)
    for comp in comps:
        inside |= comp.inside(cand)
    cand = cand[inside]
    probe = B.EvaluationPoints(cand, 3)
    B.mark_evaluation_points(sc, region, c.cache, probe)
    x = cand[~probe.download()["fallback"].astype(bool)][:24]
    assert len(x) == 24
    rounds = []
    for r in range(12):
        p = B.EvaluationPoints(x, 3)
        B.mark_evaluation_points(sc, region, c.cache, p)
        B.update_solution(sc, c.problem, region, c.cache, p, 900 + r, 0)
        rounds.append(p.solution())
    rounds = np.array(rounds)
    m_bvc = rounds.mean(0)
    se_bvc = rounds.std(0, ddof=1) / np.sqrt(len(rounds))
    est = B.wost_solve(sc, c.problem, x, B.walk_config(epsilon=c.epsilon, nWalks=32768, seed=3))
    m_w, se_w = est["mean"], est["se"]
    z = (np.abs(m_bvc - m_w) - 3e-3) / np.sqrt(se_bvc ** 2 + se_w ** 2)  # O(eps) shell allowance
    assert np.sum(z > 3.0) <= 1, (m_bvc, m_w, se_bvc, se_w)
    assert np.all(np.isfinite(m_bvc)) and np.all(se_bvc > 0)


def test_pointwise_3d_matches_harmonic_data(sphere):
    """The 3D lift of wostSolve / wostGradient / wostNormalDerivative (pointwise.h:66-76): on
    the sphere with harmonic data the estimates are unbiased for u = g, grad u = grad g and
    du/dn = n . grad g."""
    _, _, sc = sphere
    pb = B.problem(B.poisson(3), g=HARMONIC)
    rng = np.random.default_rng(4)
    x = rng.normal(size=(16, 3))
    x *= (rng.uniform(0.1, 0.7, 16) / np.linalg.norm(x, axis=1))[:, None]
    e = B.wost_solve(sc, pb, x, B.walk_config(epsilon=1e-3, nWalks=8192, seed=9))
    z = (e["mean"] - g_exact(x)) / np.maximum(e["se"], 1e-12)
    assert np.sum(np.abs(z) > 3) <= 1, z
    n = rng.normal(size=(16, 3))
    n /= np.linalg.norm(n, axis=1)[:, None]
    d = B.wost_normal_derivative(sc, pb, x, n, B.walk_config(epsilon=1e-3, nWalks=16384, seed=10))
    h = 1e-5
    dgdn = (g_exact(x + h * n) - g_exact(x - h * n)) / (2 * h)
    zd = (d["mean"] - dgdn) / np.maximum(d["se"], 1e-12)
    assert np.sum(np.abs(zd) > 3) <= 1, zd
    gr = B.wost_gradient(sc, pb, x, B.walk_config(epsilon=1e-3, nWalks=16384, seed=11))
    grad = np.stack([0.3 - x[:, 0] + x[:, 1], -0.2 - x[:, 1] + x[:, 0], 0.5 + 2 * x[:, 2]], 1)
    zg = (gr["mean"] - grad) / np.maximum(gr["se"], 1e-12)
    assert np.sum(np.abs(zg) > 3) <= 2, zg


def _cube_mesh(n=8):
    """Unit cube [0,1]^3, n x n x 2 triangles per face, outward orientation; labels: the faces
    x = 0 and x = 1 Dirichlet (0), the other four Neumann (1)."""
    V, F, L = [], [], []
    t = np.linspace(0.0, 1.0, n + 1)

    def face(origin, du, dv, label):
        base = len(V)
        for j in range(n + 1):
            for i in range(n + 1):
                V.append(origin + t[i] * du + t[j] * dv)
        for j in range(n):
            for i in range(n):
                a = base + j * (n + 1) + i
                b, c, d = a + 1, a + n + 1, a + n + 2
                F.extend([[a, b, d], [a, d, c]])  # normal du x dv
                L.extend([label, label])

    e = np.eye(3)
    face(np.zeros(3), e[2], e[1], 0)          # x = 0, normal -x
    face(e[0].copy(), e[1], e[2], 0)          # x = 1, normal +x
    face(np.zeros(3), e[0], e[2], 1)          # y = 0, normal -y
    face(e[1].copy(), e[2], e[0], 1)          # y = 1, normal +y
    face(np.zeros(3), e[1], e[0], 1)          # z = 0, normal -z
    face(e[2].copy(), e[0], e[1], 1)          # z = 1, normal +z
    V, F = np.array(V), np.array(F, np.int32)
    # weld the duplicated edge / corner vertices so that the faces share edges
    key = np.round(V * (1 << 20)).astype(np.int64)
    _, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    return V[first], inv.reshape(-1)[F].astype(np.int32), np.array(L, np.int32)


def test_screened_mixed_cube_closed_form():
    """C5's physics with a closed form: screened (sigma = 1) on the unit cube, Dirichlet
    g = e^x on x = 0 and x = 1 (linear data 1 + (e - 1) x agrees there), reflecting h = 0 on
    the other four faces: u = e^x (u'' = u, no y/z dependence). Pointwise walk-on-stars
    values and gradients, and BVC rounds, against it at |z| < 3."""
    V, F, lab = _cube_mesh(8)
    sc = B.Scene.mesh3(V, F, lab)
    pb = B.problem(B.screened(1.0, 3), g=abi.make_field(abi.FIELD_LINEAR, [np.e - 1.0, 0.0, 1.0, 0.0]))
    rng = np.random.default_rng(12)
    x = rng.uniform(0.15, 0.85, size=(24, 3))
    e = B.wost_solve(sc, pb, x, B.walk_config(epsilon=1e-3, nWalks=16384, seed=21))
    z = (e["mean"] - np.exp(x[:, 0])) / np.maximum(e["se"], 1e-12)
    assert np.all(e["se"] < 0.02) and np.sum(np.abs(z) > 3) <= 1, z
    gr = B.wost_gradient(sc, pb, x, B.walk_config(epsilon=1e-3, nWalks=32768, seed=22))
    exact = np.stack([np.exp(x[:, 0]), np.zeros(len(x)), np.zeros(len(x))], 1)
    zg = (gr["mean"] - exact) / np.maximum(gr["se"], 1e-12)
    assert np.sum(np.abs(zg) > 3) <= 2, zg
    # the cache's estimators at the region's samples, by kind (0: known Neumann, u by walks;
    # 1: offset Dirichlet patch, u and du/dn by walks), against u = e^x and du/dn = n_x e^x.
    # (The du/dn estimates are heavy-tailed where the offset patch bends down to the Neumann
    # rim and the first ball is tiny, so their mean is checked against its own standard error.)
    region = B.SolveRegion(sc, offset=0.1, epsilon=1e-3)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3, nWalks=512), nBoundary=16384, nWalksNeumann=512,
                         nWalksDirichlet=512, offset=0.1)
    c = B.generate_boundary_cache(sc, pb, region, cfg, 7, 0).download()
    kinds = region.kinds[c["segment"]]
    ux = np.exp(c["z"][:, 0])
    dx = c["n"][:, 0] * ux
    assert set(np.unique(kinds)) == {0, 1}
    for k in (0, 1):
        m = kinds == k
        eu = c["uHat"][m] - ux[m]
        assert abs(eu.mean()) <= 4 * eu.std(ddof=1) / np.sqrt(m.sum()) + 2e-3, (k, eu.mean())  # O(eps) shell
        ed = c["dHat"][m] - dx[m]
        assert abs(ed.mean()) <= 5 * ed.std(ddof=1) / np.sqrt(m.sum()) + 1e-6, (k, ed.mean())
    assert np.all(c["dHat"][kinds == 0] == 0.0)  # h = 0 is data there
    assert abs(np.mean(1.0 / c["pdf"]) - 6.24) < 0.05  # the region surface's area
    # the representation itself: the gather over this sample set with the exact u and du/dn
    # reproduces e^x (quadrature error of 16384 samples), and with the walks' u as well
    xi = rng.uniform(0.2, 0.8, size=(512, 3))
    spec = B.make_splat_config(sc, pb, cfg)
    for uh in (ux, c["uHat"]):
        cache = B.BoundaryCache.from_arrays(c["z"], c["n"], c["pdf"], uh, dx, segment=c["segment"])
        p = B.EvaluationPoints(xi, 3)
        B.splat_solution(cache, None, p, spec)
        err = p.solution() - np.exp(xi[:, 0])
        assert np.sqrt(np.mean(err ** 2)) < 6e-3 and abs(err.mean()) < 3e-3, (err.mean(), np.sqrt(np.mean(err ** 2)))


def test_3d_walks_reject_neumann_data_and_sources():
    """What the 3D walks do not implement fails loudly instead of being dropped: nonzero
    Neumann data h (the ball-clipped neumannTerm of pointwise.cpp:52-107 is 2D) and source
    terms f (sampleBallGreens, kernels.cpp:98-99, is 2D-only); h = 0 as data is accepted."""
    V, F, lab = _cube_mesh(4)
    sc = B.Scene.mesh3(V, F, lab)
    g = abi.make_field(abi.FIELD_LINEAR, [1.0, 0.0, 0.0, 0.0])
    x = np.array([[0.5, 0.5, 0.5]])
    wc = B.walk_config(epsilon=1e-3, nWalks=64, seed=1)
    with pytest.raises(B.SolverError, match="Neumann data"):
        B.wost_solve(sc, B.problem(B.poisson(3), g=g, h=abi.make_field(abi.FIELD_CONSTANT, [1.0])), x, wc)
    with pytest.raises(B.SolverError, match="source terms"):
        B.wost_solve(sc, B.problem(B.poisson(3), g=g, f=abi.make_field(abi.FIELD_CONSTANT, [1.0])), x, wc)
    e = B.wost_solve(sc, B.problem(B.poisson(3), g=g, h=abi.make_field(abi.FIELD_CONSTANT, [0.0])), x, wc)
    assert np.isfinite(e["mean"][0]) and abs(e["mean"][0] - 0.5) < 0.2  # u = x with reflecting side faces
