"""Walk parity at BASELINE's own configurations (C1-C3, full geometry and walk
parameters): the cache's per-sample estimates against the reference's wostSolve /
wostNormalDerivative (pointwise.cpp:233-288, oracle/_ref) at the GPU's own sample
positions, plus the port of the reference's full-pipeline test
(test_cache.cpp:961-993).

Per sample and estimator, z = (m_gpu - m_ref) / sqrt(se_gpu^2 + se_ref^2), with
4096 walks on each side. The cache itself does not keep per-sample standard errors
(cache.cpp:337,344,350 drop them, as the GPU cache does), so se_gpu comes from an
independent 4096-walk GPU re-estimate at the same position. With ~400 z-scores per
config, |z| > 3 happens by chance at rate 0.27%: the test allows the binomial
99.99% quantile of that count."""
import concurrent.futures as cf
import os

import numpy as np
import pytest
from scipy import stats

import paper_2302_11825_b200 as B
from oracle import oracle as O
from paper_2302_11825_b200 import abi, configs
from tests import helpers as H

pytestmark = [pytest.mark.gpu, pytest.mark.ref]

WALKS = 4096
SHARDS = 8        # sample ranges spread around the boundary
PER_SHARD = 25    # 8 x 25 = 200 samples per config


def _build(cid):
    c = configs.CONFIGS[cid]()
    sc = B.Scene(c.vertices, c.segments, c.labels)
    rs = O.RefScene(c.vertices, c.segments, c.labels)
    if c.region_mode == abi.REGION_SUBDOMAIN:
        sub = B.Scene(c.sub_vertices, c.sub_segments, np.zeros(len(c.sub_segments), np.int32))
        region = B.SolveRegion(sc, abi.REGION_SUBDOMAIN, c.region_offset, sub, epsilon=c.epsilon)
    else:
        region = B.SolveRegion(sc, offset=c.region_offset, epsilon=c.epsilon)
    return c, sc, rs, region


def _binomial_cap(n, p=0.0027, q=1e-4):
    return int(stats.binom.isf(q, n, p))


def _ref_map(fn, items):
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:  # ctypes releases the GIL
        return list(ex.map(fn, items))


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_cache_estimates_vs_reference_at_config(cid):
    c, sc, rs, region = _build(cid)
    cfg = c.cache
    N = cfg.nBoundary
    cfg.nWalksNeumann = cfg.nWalksDirichlet = WALKS
    # the cache's own samples: contiguous ranges of the full-N stratified positions
    parts = []
    for k in range(SHARDS):
        lo = (k * N) // SHARDS
        parts.append(B.generate_boundary_cache(sc, c.problem, region, cfg, c.seed, 3, begin=lo,
                                               end=lo + PER_SHARD).download())
    cache = {key: np.concatenate([p[key] for p in parts]) for key in ("z", "n", "uHat", "dHat", "segment")}
    kinds = region.kinds[cache["segment"]]
    known = kinds == abi.SEG_KNOWN_NEUMANN
    z, n = cache["z"], cache["n"]
    x_u = np.where(known[:, None], z - 0.5 * c.epsilon * n, z)  # cache.cpp:329-339
    wc = B.walk_config(epsilon=c.epsilon, nWalks=WALKS, seed=c.seed + 101)
    g_u = B.wost_solve(sc, c.problem, x_u, wc)
    est = ~known
    g_d = B.wost_normal_derivative(sc, c.problem, z[est], n[est], wc)
    rwc = abi.default_walk_config()
    rwc.epsilon, rwc.nWalks = c.epsilon, WALKS

    def ref_u(i):
        w = abi.WalkConfig.from_buffer_copy(rwc)
        w.seed = 5000 + i
        return rs.solve(c.problem, x_u[i], w, 1)

    def ref_d(i):
        w = abi.WalkConfig.from_buffer_copy(rwc)
        w.seed = 9000 + i
        return rs.gradient(c.problem, z[i], w, normal=n[i])

    ru = _ref_map(ref_u, range(len(z)))
    idx_d = np.flatnonzero(est)
    rd = _ref_map(ref_d, idx_d)
    zs = [H.zscore(cache["uHat"][i], g_u["se"][i], ru[i][0], ru[i][1]) for i in range(len(z))]
    zs += [H.zscore(cache["dHat"][i], g_d["se"][j], rd[j][0], rd[j][1]) for j, i in enumerate(idx_d)]
    zs = np.abs(np.array(zs))
    assert np.all(np.isfinite(zs))
    # KnownNeumann samples carry d = h(z) exactly (cache.cpp:329-339)
    assert np.all(cache["dHat"][known] == 0.0)
    cap = _binomial_cap(len(zs))
    assert np.sum(zs > 3) <= cap, (np.sum(zs > 3), cap, np.sort(zs)[-5:])
    # and no systematic offset: the mean z is within 4 / sqrt(n) of 0
    zsig = [H.zscore(cache["uHat"][i], g_u["se"][i], ru[i][0], ru[i][1]) for i in range(len(z))]
    assert abs(np.mean(zsig)) < 4 / np.sqrt(len(zsig)), np.mean(zsig)


@pytest.mark.parametrize("name,maker,x,exact", [("disk-linear", H.disk_linear, (0.4, 0.2), 0.4),
                                                ("square-mixed-linear", H.square_mixed, (0.3, 0.6), 0.3),
                                                ("screened-constant", H.screened_constant, (0.7, 0.4), 1.0)])
def test_full_pipeline_matches_closed_forms_48_seeds(name, maker, x, exact):
    """test_cache.cpp:961-993 ("full pipeline matches closed forms at matched statistics"),
    plain mode: the default whole-domain region (l = 5 eps, eps = 1e-3 diag), N = M = 64,
    16 / 64 walks, seeds 1000..1047; |mean - exact| <= 4 se over the 48 rounds."""
    geom, pb = maker()
    sc = B.Scene(*geom)
    region = B.SolveRegion(sc, epsilon=1e-3 * sc.diagonal)
    cfg = B.cache_config(nBoundary=64, nSource=64, nWalksNeumann=16, nWalksDirichlet=64)
    vals = []
    for seed in range(48):
        pts = B.EvaluationPoints([x])
        B.mark_evaluation_points(sc, region, cfg, pts)
        assert not pts.download()["fallback"][0]
        B.update_solution(sc, pb, region, cfg, pts, 1000 + seed, 0)
        vals.append(pts.solution()[0])
    vals = np.array(vals)
    m, se = vals.mean(), vals.std(ddof=1) / np.sqrt(len(vals))
    assert abs(m - exact) <= 4.0 * se, (m, se)
