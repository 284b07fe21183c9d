"""Clamped and ball-kernel splats on the GPU: correctedBoundarySplat
cache.cpp:499-553, correctedSourceSplat 555-597, the mode dispatch of updateSolution
639-662 and markEvaluationPoints' ball radius 268-274. Mirrors test_cache.cpp:748-959:
the deterministic loops against the reference's outputs on identical caches
(tests/golden/clamp.npz), the sampled corrections statistically against closed forms."""
import math

import numpy as np
import pytest

import paper_2302_11825_b200 as B
from oracle import oracle as O
from paper_2302_11825_b200 import abi
from tests import helpers as H

pytestmark = pytest.mark.gpu

DIAG = 2.0 * math.sqrt(2.0)  # unit 256-gon bounding-box diagonal


def circle():
    v, s, lab = O.circle_geometry(segments=256)
    sc = B.Scene(v, s, lab)
    region = B.SolveRegion(sc, mode=abi.REGION_SUBDOMAIN, subdomain=B.Scene(v, s, lab))  # loopRegion(circle)
    return v, s, sc, region


def plain_cfg(ball=False, kernel=None):
    k = kernel or H.kspec(0, 0, 2, DIAG)
    return abi.SplatConfig(abi.KernelSpec(k.kind, k.sigma, 2, DIAG), 1e-12 * DIAG, 0, int(ball))


def exact_boundary_cache(v, s, n, seed, u, d):
    """exactBoundaryCache: uniform arc-length samples with exact data (pdf 1/L)."""
    rng = np.random.default_rng(seed)
    a, b = v[s[:, 0]], v[s[:, 1]]
    ln = np.linalg.norm(b - a, axis=1)
    L = ln.sum()
    seg = rng.choice(len(s), size=n, p=ln / L)
    t = rng.uniform(size=n)
    z = a[seg] + t[:, None] * (b[seg] - a[seg])
    e = (b - a)[seg] / ln[seg][:, None]
    nrm = np.stack([e[:, 1], -e[:, 0]], 1)
    return B.BoundaryCache.from_arrays(z, nrm, np.full(n, 1.0 / L), u(z), d(z, nrm))


def exact_source_cache(v, m, seed, f):
    """exactSourceCache: uniform samples in the polygon (pdf 1/area)."""
    rng = np.random.default_rng(seed)
    area = 0.5 * np.sum(v[:, 0] * np.roll(v[:, 1], -1) - np.roll(v[:, 0], -1) * v[:, 1])
    ys = []
    sc = O.OracleScene(v, np.stack([np.arange(len(v)), (np.arange(len(v)) + 1) % len(v)], 1).astype(np.int32),
                       np.zeros(len(v), np.int32))
    while sum(len(y) for y in ys) < m:
        c = rng.uniform(-1, 1, (2 * m, 2))
        ys.append(c[sc.inside(c)])
    y = np.concatenate(ys)[:m]
    return B.SourceCache.from_arrays(y, np.full(m, 1.0 / area), f(y))


def mean_se(vals):
    vals = np.asarray(vals)
    return vals.mean(), vals.std(ddof=1) / math.sqrt(len(vals))


def ball_points(sc, region, x):
    pts = B.EvaluationPoints(np.atleast_2d(x))
    B.mark_evaluation_points(sc, region, B.cache_config(sourceBall=1), pts)
    return pts


# --- deterministic loops vs the reference ---------------------------------------------

def test_clamped_and_ball_splats_match_reference(golden):
    g = golden("clamp")
    v, s, sc, region = circle()
    bc = B.BoundaryCache.from_arrays(g["b_z"], g["b_n"], g["b_pdf"], g["b_uHat"], g["b_dHat"])
    scc = B.SourceCache.from_arrays(g["s_y"], g["s_pdf"], g["s_f"])
    # markEvaluationPoints' ball radius on the GPU equals the reference's
    pts = ball_points(sc, region, g["x"])
    np.testing.assert_allclose(pts.download()["ballRadius"], g["ballRadius"], rtol=1e-14)
    for i, (mode, c) in enumerate(g["cases"]):
        mode, c = int(mode), float(c)
        ball = bool(mode & 2)
        cfg = plain_cfg(ball)
        p = ball_points(sc, region, g["x"]) if ball else B.EvaluationPoints(g["x"])
        if mode & 1:
            B.corrected_boundary_splat(bc, p, region, cfg, c, abi.CLAMP_ONLY)
        else:
            B.splat_solution(bc, None, p, cfg)
        if mode & 4:
            B.corrected_source_splat(scc, p, region, cfg, c)
        else:
            B.splat_solution(None, scc, p, cfg)
        st = p.download()
        for key in ("boundarySum", "sourceSum"):
            assert H.rel_err(st[key], g[f"{i}_{key}"]) < 1e-4, (i, mode, key, H.rel_err(st[key], g[f"{i}_{key}"]))
        for key in ("nBoundary", "mSource", "skipped"):
            assert np.array_equal(st[key], g[f"{i}_{key}"]), (i, key)


def test_infinite_bound_reproduces_plain_splat():
    """test_cache.cpp:748-764: bit-identical sums."""
    v, s, sc, region = circle()
    bc = exact_boundary_cache(v, s, 256, 61, lambda z: z[:, 0], lambda z, n: n[:, 0])
    x = [[0.9, 0.0], [0.2, 0.1]]
    a, b = B.EvaluationPoints(x), B.EvaluationPoints(x)
    B.splat_solution(bc, None, a, plain_cfg())
    B.corrected_boundary_splat(bc, b, region, plain_cfg(), math.inf, abi.CLAMP_ONLY)
    sa, sb = a.download(), b.download()
    assert np.array_equal(sa["boundarySum"], sb["boundarySum"])
    assert np.array_equal(sa["nBoundary"], sb["nBoundary"])


def clamped_winding_quad(v, s, x, c, sub=256):
    """clampedWindingQuad: midpoint quadrature of the clamped Poisson kernel over the polygon."""
    a, b = v[s[:, 0]], v[s[:, 1]]
    t = (np.arange(sub) + 0.5) / sub
    tot = 0.0
    for k in range(len(s)):
        e = b[k] - a[k]
        ln = np.linalg.norm(e)
        n = np.array([e[1], -e[0]]) / ln
        z = a[k] + t[:, None] * e
        dz = z - x
        P = dz @ n / (2 * np.pi * np.sum(dz * dz, 1))
        tot += np.sum(np.clip(P, -c, c)) * ln / sub
    return tot


def test_clamping_bias_and_ray_correction():
    """test_cache.cpp:766-809."""
    v, s, sc, region = circle()
    x = np.array([0.95, 0.0])
    a, b = v[s[:, 0]], v[s[:, 1]]
    mid = 0.5 * (a + b)
    e = b - a
    n = np.stack([e[:, 1], -e[:, 0]], 1) / np.linalg.norm(e, axis=1)[:, None]
    mags = np.sort(np.abs(np.sum((mid - x) * n, 1) / (2 * np.pi * np.sum((mid - x) ** 2, 1))))
    c = mags[len(mags) * 3 // 4]
    assert np.mean(mags > c) >= 0.2
    target = clamped_winding_quad(v, s, x, c)
    assert abs(target - 1.0) > 1e-3
    one = B.field_evaluator(abi.make_field(abi.FIELD_CONSTANT, [1.0]))
    clamp_only, corrected = [], []
    for seed in range(300):
        bc = exact_boundary_cache(v, s, 128, 6700 + seed, lambda z: np.ones(len(z)), lambda z, n: np.zeros(len(z)))
        p = B.EvaluationPoints([x])
        B.corrected_boundary_splat(bc, p, region, plain_cfg(), c, abi.CLAMP_ONLY, None, seed, 1)
        clamp_only.append(p.solution()[0])
        q = B.EvaluationPoints([x])
        B.corrected_boundary_splat(bc, q, region, plain_cfg(), c, abi.CLAMP_CORRECT, one, seed, 2)
        corrected.append(q.solution()[0])
    mo, so = mean_se(clamp_only)
    mc, sc_ = mean_se(corrected)
    assert abs(mo - target) <= 4 * so, (mo, target, so)
    assert abs(mo - 1.0) > 5 * so
    assert abs(mc - 1.0) <= 3 * sc_, (mc, sc_)


def test_correction_alone_recovers_winding_number():
    """test_cache.cpp:811-832: at c -> 0 the ray correction carries the whole integral."""
    v, s, sc, region = circle()
    one = B.field_evaluator(abi.make_field(abi.FIELD_CONSTANT, [1.0]))
    ins, out = [], []
    for seed in range(300):
        bc = exact_boundary_cache(v, s, 64, 7100 + seed, lambda z: np.ones(len(z)), lambda z, n: np.zeros(len(z)))
        p = B.EvaluationPoints([[0.4, -0.1], [2.0, 0.3]])
        B.corrected_boundary_splat(bc, p, region, plain_cfg(), 1e-9, abi.CLAMP_CORRECT, one, seed, 3)
        u = p.solution()
        ins.append(u[0])
        out.append(u[1])
    mi, si = mean_se(ins)
    mo, so = mean_se(out)
    assert abs(mi - 1.0) <= max(3 * si, 1e-6), (mi, si)
    assert abs(mo) <= max(4 * so, 1e-6), (mo, so)


def test_clamped_splat_argument_validation():
    """test_cache.cpp:834-851."""
    v, s, sc, region = circle()
    bc = exact_boundary_cache(v, s, 16, 73, lambda z: np.ones(len(z)), lambda z, n: np.zeros(len(z)))
    p = B.EvaluationPoints([[0.0, 0.0]])
    with pytest.raises(B.InvalidArgument):
        B.corrected_boundary_splat(bc, p, region, plain_cfg(), 1.0, abi.CLAMP_OFF)
    with pytest.raises(B.InvalidArgument):
        B.corrected_boundary_splat(bc, p, region, plain_cfg(), -1.0, abi.CLAMP_ONLY)
    with pytest.raises(B.InvalidArgument):
        B.corrected_boundary_splat(bc, p, region, plain_cfg(), 1.0, abi.CLAMP_CORRECT)
    # ball mode without marked radii (requireBallRadius cache.cpp:418-423)
    with pytest.raises(B.SolverError):
        B.splat_solution(bc, None, p, plain_cfg(ball=True))


# --- ball-kernel source mode (test_cache.cpp:853-959) ---------------------------------

def test_ball_source_infinite_bound_integrates_the_source():
    v, s, sc, region = circle()
    one = abi.make_field(abi.FIELD_CONSTANT, [1.0])
    vals = []
    for seed in range(200):
        scc = exact_source_cache(v, 256, 8300 + seed, lambda y: np.ones(len(y)))
        p = ball_points(sc, region, [0.0, 0.0])
        assert abs(p.download()["ballRadius"][0] - 1.0) < 1e-3
        B.corrected_source_splat(scc, p, region, plain_cfg(ball=True), math.inf, one, seed, 4)
        vals.append(p.solution()[0])
    m, se = mean_se(vals)
    assert abs(m + 0.25) <= 4 * max(se, 1e-6), (m, se)


def test_ball_kernel_suppresses_the_normal_derivative_term():
    v, s, sc, region = circle()
    bc1 = exact_boundary_cache(v, s, 64, 87, lambda z: np.zeros(len(z)), lambda z, n: np.full(len(z), 0.5))
    d1 = bc1.download()
    bc2 = B.BoundaryCache.from_arrays(d1["z"], d1["n"], d1["pdf"], d1["uHat"], np.full(64, 123.0))
    p1, p2 = ball_points(sc, region, [0.0, 0.0]), ball_points(sc, region, [0.0, 0.0])
    B.splat_solution(bc1, None, p1, plain_cfg(ball=True))
    B.splat_solution(bc2, None, p2, plain_cfg(ball=True))
    assert abs(p1.solution()[0] - p2.solution()[0]) < 0.01


def test_ball_source_zero_field_and_vanishing_bound():
    v, s, sc, region = circle()
    zero = abi.make_field(abi.FIELD_CONSTANT, [0.0])
    zc = exact_source_cache(v, 64, 89, lambda y: np.zeros(len(y)))
    p = ball_points(sc, region, [0.1, 0.2])
    B.corrected_source_splat(zc, p, region, plain_cfg(ball=True), 1e-6, zero, 0, 5)
    assert p.download()["sourceSum"][0] == 0.0
    # c -> 0: the ball-sampled correction alone carries int G^B f
    fvar = abi.make_field(abi.FIELD_QUADRATIC3, [2.0, 0, 0, 0, 1.0, 0, 0, 0, 0, 0])
    target = -0.5 - 1.0 / 32.0  # 2 * mass(1) + int_0^1 (ln r / 2 pi) r^2 r dr * pi
    vals = []
    for seed in range(400):
        scc = exact_source_cache(v, 128, 9100 + seed, lambda y: 2.0 + y[:, 0] ** 2)
        q = ball_points(sc, region, [0.0, 0.0])
        B.corrected_source_splat(scc, q, region, plain_cfg(ball=True), 1e-12, fvar, seed, 6)
        vals.append(q.solution()[0])
    m, se = mean_se(vals)
    assert abs(m - target) <= 4 * se, (m, target, se)


def test_ball_source_update_solution_end_to_end():
    geom, pb = H.disk_poisson()
    sc = B.Scene(*geom)
    region = B.SolveRegion(sc, epsilon=1e-3 * sc.diagonal)
    cfg = B.cache_config(sourceBall=1, nBoundary=64, nSource=128, nWalksNeumann=16, nWalksDirichlet=16)
    vals = []
    for seed in range(48):
        p = B.EvaluationPoints([[0.0, 0.0]])
        B.mark_evaluation_points(sc, region, cfg, p)
        assert not p.download()["fallback"][0]
        B.update_solution(sc, pb, region, cfg, p, 500 + seed, 0)
        vals.append(p.solution()[0])
    m, se = mean_se(vals)
    assert abs(m + 0.25) <= 4 * se, (m, se)
    # ball mode rejects non-Poisson kernels and gradient requests
    p = ball_points(sc, region, [0.0, 0.0])
    scc = exact_source_cache(geom[0], 8, 93, lambda y: np.ones(len(y)))
    with pytest.raises(B.SolverError):
        B.corrected_source_splat(scc, p, region, plain_cfg(ball=True, kernel=H.kspec(1, 1.0)), 1.0,
                                 abi.make_field(abi.FIELD_CONSTANT, [1.0]))
    whole = B.SolveRegion(sc, offset=0.05, epsilon=1e-3)
    gcfg = B.cache_config(sourceBall=1, offset=0.05)
    g = B.EvaluationPoints([[0.0, 0.0]])
    B.mark_evaluation_points(sc, whole, gcfg, g)
    with pytest.raises(B.SolverError):
        B.update_solution(sc, pb, whole, gcfg, g, 0, 0, gradients=True)


# --- clamp modes through updateSolution (cache.cpp:648-661) ---------------------------

@pytest.mark.parametrize("mode", [abi.CLAMP_ONLY, abi.CLAMP_CORRECT])
def test_update_solution_clamp_modes(mode):
    """Near-boundary point of disk-linear with a tight bound: ClampCorrect (default walk
    evaluator) stays unbiased, ClampOnly carries the clamping bias."""
    geom, pb = H.disk_linear()
    sc = B.Scene(*geom)
    region = B.SolveRegion(sc, epsilon=1e-3 * sc.diagonal)
    x = np.array([[0.9, 0.1]])
    cfg = B.cache_config(clampMode=mode, clamp=0.5, nBoundary=256, nWalksNeumann=16, nWalksDirichlet=64,
                         correctionWalks=4)
    vals = []
    for seed in range(64):
        p = B.EvaluationPoints(x)
        B.mark_evaluation_points(sc, region, cfg, p)
        B.update_solution(sc, pb, region, cfg, p, 2000 + seed, 0, gradients=True)
        st = p.download()
        assert st["nBoundaryGrad"][0] == 256  # the gradient splat is unclamped and still runs
        vals.append(p.solution(st)[0])
    m, se = mean_se(vals)
    if mode == abi.CLAMP_CORRECT:
        assert abs(m - 0.9) <= 4 * se, (m, se)
    else:
        assert abs(m - 0.9) > 4 * se, (m, se)


def test_update_solution_correction_evaluator():
    """updateSolution's correctionEval argument (cache.h:195-198, cache.cpp:646-648): an
    explicit walk evaluator equals the empty default bit for bit (makeDefaultEvaluator,
    cache.cpp:600-620); an exact-data evaluator (u = x on disk-linear) replaces the
    correction walks and stays unbiased."""
    geom, pb = H.disk_linear()
    sc = B.Scene(*geom)
    region = B.SolveRegion(sc, epsilon=1e-3 * sc.diagonal)
    x = np.array([[0.9, 0.1], [0.5, -0.3]])
    # a bound tight enough that both points' rays have saturated crossings every round
    cfg = B.cache_config(clampMode=abi.CLAMP_CORRECT, clamp=0.05, nBoundary=256, nWalksNeumann=16,
                         nWalksDirichlet=64, correctionWalks=4)

    def run(ev, seed):
        p = B.EvaluationPoints(x)
        B.mark_evaluation_points(sc, region, cfg, p)
        B.update_solution(sc, pb, region, cfg, p, 3000 + seed, 0, correction_eval=ev)
        return p.download()

    a, b = run(None, 0), run(B.walk_evaluator(sc, pb, cfg), 0)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    none = abi.BoundaryEvaluator()  # kind NONE = the empty std::function = the default
    c = run(none, 0)
    for k in a:
        np.testing.assert_array_equal(a[k], c[k], err_msg=k)
    exact = B.field_evaluator(abi.make_field(abi.FIELD_LINEAR, [1, 0, 0, 0]))
    d = run(exact, 0)
    assert not np.array_equal(a["boundarySum"], d["boundarySum"])  # the correction used the field
    vals = [run(exact, seed) for seed in range(48)]
    m, se = mean_se([st["boundarySum"][0] / st["nBoundary"][0] for st in vals])
    assert abs(m - 0.9) <= 4 * se, (m, se)
