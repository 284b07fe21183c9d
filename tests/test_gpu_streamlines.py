"""Streamlines (runStreamlines tools/src/runner.cpp:285-373) on the GPU: all seeds
advance together, two batched gradient gathers per Heun step over retained caches.
Pinned against the tracing loop restated over the reference's own Scene::inside,
markEvaluationPoints and splatGradient on the identical (downloaded) caches."""
import numpy as np
import pytest

import paper_2302_11825_b200 as B
from oracle import oracle as O
from tests import helpers as H

pytestmark = pytest.mark.gpu


def _setup(maker, **kw):
    geom, pb = maker()
    sc = B.Scene(*geom)
    region = B.SolveRegion(sc, offset=0.05, epsilon=1e-3)
    cfg = B.cache_config(B.walk_config(epsilon=1e-3), offset=0.05, **kw)
    return geom, pb, sc, region, cfg


def test_streamlines_match_reference_loop_on_identical_caches():
    geom, pb, sc, region, cfg = _setup(H.disk_poisson, nBoundary=256, nSource=256, nWalksNeumann=32,
                                       nWalksDirichlet=64)
    seeds = np.array([[0.3, 0.1], [-0.2, -0.4], [0.0, 0.6], [3.0, 0.0], [0.05, -0.02]])
    rounds, h, steps = 2, 0.05, 30
    gpu = B.trace_streamlines(sc, pb, region, cfg, 7, rounds, seeds, h, steps)
    caches = []
    for r in range(rounds):
        bc = B.generate_boundary_cache(sc, pb, region, cfg, 7, r).download()
        sc_ = B.generate_source_cache(pb, region, cfg, 7, r).download()
        caches.append((bc, sc_))
    rs = O.RefScene(*geom)
    rr = O.RefRegion(rs, offset=0.05, eps=1e-3)
    spec = H.kspec(0, 0, 2, rs.diagonal)
    ref_lines, ref_reasons = O.ref_streamlines(rs, rr, cfg, spec, 1e-12 * rs.diagonal, caches, seeds, h, steps)
    assert gpu["reasons"] == ref_reasons, (gpu["reasons"], ref_reasons)
    for a, b in zip(gpu["polylines"], ref_lines):
        assert a.shape == b.shape
        np.testing.assert_allclose(a, b, atol=2e-5)
    # the seed outside the disk has no polyline; radial flow (grad u = x / 2) leaves the region
    assert gpu["counts"][3] == 0 and gpu["reasons"][3] == "outside"
    for line in gpu["polylines"][:3]:
        r = np.linalg.norm(line, axis=1)
        assert np.all(np.diff(r) > 0) and r[-1] > 0.85


def test_streamlines_linear_field_and_validation():
    geom, pb, sc, region, cfg = _setup(H.disk_linear, nBoundary=1024, nWalksNeumann=64, nWalksDirichlet=256)
    out = B.trace_streamlines(sc, pb, region, cfg, 3, 2, [[-0.5, 0.2], [0.0, -0.3]], 0.02, 200)
    for line, reason in zip(out["polylines"], out["reasons"]):
        assert reason == "outside"
        # away from the region boundary (within a few sample spacings of the cache
        # the splatted gradient is heavy-tailed and the Heun average may shorten)
        steps = np.diff(line, axis=0)[np.linalg.norm(line[1:], axis=1) < 0.85]
        assert len(steps) > 20
        assert np.all(np.abs(np.linalg.norm(steps, axis=1) - 0.02) < 2e-3)  # unit direction, step h
        assert np.all(steps[:, 0] > 0.015)  # grad u = (1, 0)
        assert np.max(np.abs(line[:, 1] - line[0, 1])) < 0.05
        assert line[-1, 0] > 0.8
    with pytest.raises(B.InvalidArgument):
        B.trace_streamlines(sc, pb, region, cfg, 3, 1, [[0.0, 0.0]], -1.0, 10)
    ball = B.cache_config(sourceBall=1, offset=0.05)
    with pytest.raises(B.InvalidArgument):
        B.trace_streamlines(sc, pb, region, ball, 3, 1, [[0.0, 0.0]], 0.1, 10)
