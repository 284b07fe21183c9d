"""Host-side logic of the product (C++ in libbvc_b200.so, runs without a GPU):
Scene::build semantics and buildSolveRegion (cache.cpp:137-246), checked against
the reference's own outputs (tests/golden/regions.npz and oracle/_ref)."""
import numpy as np
import pytest

import paper_2302_11825_b200 as B
from oracle import oracle as O
from paper_2302_11825_b200 import abi, configs
from tests import helpers as H


@pytest.mark.parametrize("name", ["square_d", "square_mixed", "disk", "annulus", "star"])
def test_region_matches_reference(golden, name):
    g = golden("regions")
    sc = B.Scene(g[name + "_in_v"], g[name + "_in_s"], g[name + "_in_lab"])
    r = B.SolveRegion(sc, abi.REGION_WHOLE_DOMAIN, float(g[name + "_offset"][0]), epsilon=1e-3)
    np.testing.assert_allclose(r.vertices, g[name + "_v"], rtol=0, atol=1e-13)
    assert np.array_equal(r.segments, g[name + "_s"])
    assert np.array_equal(r.labels, g[name + "_lab"])
    assert np.array_equal(r.kinds, g[name + "_kinds"])
    assert np.array_equal(r.source, g[name + "_src"])
    assert r.area == pytest.approx(float(g[name + "_area"][0]), rel=1e-12)


def test_square_region_shrinks_by_offset():
    """test_cache.cpp:107-122: all-Dirichlet square, l = 0.1 -> area 0.64; default l = 5 eps."""
    v, s, lab = O.rectangle_geometry([0, 0], [1, 1], [0, 0, 0, 0])
    sc = B.Scene(v, s, lab)
    r = B.SolveRegion(sc, offset=0.1, epsilon=1e-3)
    assert r.whole_domain and r.offset == 0.1 and r.area == pytest.approx(0.64, rel=1e-12)
    assert r.boundary.lo[0] == pytest.approx(0.1) and r.boundary.hi[1] == pytest.approx(0.9)
    assert np.all(r.kinds == abi.SEG_ESTIMATED_OFFSET)
    assert B.SolveRegion(sc, epsilon=1e-3).offset == pytest.approx(5e-3)


def test_region_errors_match_reference():
    # offset must exceed epsilon (cache.cpp:139)
    v, s, lab = O.rectangle_geometry([0, 0], [1, 1], [0, 0, 0, 0])
    with pytest.raises(B.InvalidArgument):
        B.SolveRegion(B.Scene(v, s, lab), offset=1e-3, epsilon=1e-3)
    # BASELINE config 2 at l = 5 eps: the reference throws ParseError too (see configs.py)
    c = configs.config2()
    with pytest.raises(B.ParseError, match="inverted"):
        B.SolveRegion(B.Scene(c.vertices, c.segments, c.labels), offset=0.0, epsilon=1e-3)
    r = B.SolveRegion(B.Scene(c.vertices, c.segments, c.labels), offset=c.region_offset, epsilon=1e-3)
    assert r.area == pytest.approx(2 * (2 - 2 * c.region_offset), rel=1e-12)


@pytest.mark.ref
def test_config2_region_matches_reference_and_c2_l5eps_throws():
    c = configs.config2()
    rs = O.RefScene(c.vertices, c.segments, c.labels)
    with pytest.raises(ValueError, match="inverted"):
        O.RefRegion(rs, abi.REGION_WHOLE_DOMAIN, 0.0, eps=1e-3)
    rr = O.RefRegion(rs, abi.REGION_WHOLE_DOMAIN, c.region_offset, eps=1e-3)
    r = B.SolveRegion(B.Scene(c.vertices, c.segments, c.labels), offset=c.region_offset, epsilon=1e-3)
    np.testing.assert_allclose(r.vertices, rr.vertices, atol=1e-13)
    assert np.array_equal(r.kinds, rr.kinds)


def test_subdomain_region_passes_loop_through():
    v, s, lab = O.circle_geometry(segments=64)
    sub = B.Scene(*O.circle_geometry(radius=0.5, segments=32))
    r = B.SolveRegion(B.Scene(v, s, lab), abi.REGION_SUBDOMAIN, 0.01, subdomain=sub, epsilon=1e-3)
    assert not r.whole_domain and np.all(r.kinds == abi.SEG_USER_LOOP) and np.all(r.source == -1)
    assert r.area == pytest.approx(O.OracleScene(*O.circle_geometry(radius=0.5, segments=32)).area(), rel=1e-12)
    cw = B.Scene(*O.circle_geometry(radius=0.5, segments=32, ccw=False))
    with pytest.raises(B.ParseError):
        B.SolveRegion(B.Scene(v, s, lab), abi.REGION_SUBDOMAIN, 0.01, subdomain=cw, epsilon=1e-3)


def test_scene_build_validation():
    """Scene::build error cases (scene.cpp:11-51)."""
    v = np.array([[0, 0], [1, 0], [0, 1]], float)
    with pytest.raises(B.ParseError, match="out-of-range"):
        B.Scene(v, [[0, 1], [1, 5]], [0, 0])
    with pytest.raises(B.ParseError, match="zero length"):
        B.Scene(np.array([[0, 0], [0, 0], [1, 1]], float), [[0, 1], [1, 2], [2, 0]], [0, 0, 0])
    with pytest.raises(B.ParseError, match="non-manifold"):
        B.Scene(v, [[0, 1], [0, 2], [1, 2]], [0, 0, 0])
    open_chain = B.Scene(v, [[0, 1], [1, 2]], [1, 1])
    assert not open_chain.closed and open_chain.has_neumann()
    sc = B.Scene(*O.circle_geometry(segments=16))
    assert sc.closed and sc.n_loops == 1 and sc.diagonal == pytest.approx(np.hypot(2, 2), rel=1e-12)


def test_configs_shapes():
    c1 = configs.config1()
    assert len(c1.points) == 46112 and len(c1.segments) == 1024 and c1.cache.nBoundary == 4096
    c2 = configs.config2()
    assert len(c2.points) == 512 * 512 and len(c2.segments) == 2048 and c2.cache.nBoundary == 16384
    c3 = configs.config3(grid_n=64)
    assert len(c3.segments) == 16384 and c3.cache.nSource == 65536 and c3.problem.kernel.sigma == 10.0
