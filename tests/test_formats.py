"""The data formats either side of the path, host code behind the C ABI:
GridField CSV (grid.cpp:22-96), the PGM view (tools/src/image.cpp:12-51) and the
streamline CSV (runner.cpp:333-369). No GPU needed."""
import numpy as np
import pytest

import paper_2302_11825_b200 as B
from oracle import oracle as O


def _grid(seed=0, nx=7, ny=5):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(ny, nx)) * 10.0 ** rng.integers(-8, 8, size=(ny, nx))
    ok = rng.uniform(size=(ny, nx)) > 0.2
    return (-1.25, 0.5), 0.125, v, ok


def test_grid_csv_round_trip(tmp_path):
    origin, h, v, ok = _grid()
    p = tmp_path / "g.csv"
    B.save_grid_csv(p, origin, h, v, ok)
    o2, h2, v2, ok2 = B.load_grid_csv(p)
    assert o2 == origin and h2 == h
    assert np.array_equal(v2, v) and np.array_equal(ok2, ok)  # %.17g round-trips exactly
    lines = p.read_text().splitlines()
    assert lines[0] == "x,y,value,valid" and len(lines) == 1 + v.size


@pytest.mark.ref
def test_grid_csv_matches_reference_bytes_and_rmse(tmp_path):
    origin, h, v, ok = _grid(1)
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    B.save_grid_csv(a, origin, h, v, ok)
    O.ref_grid_save_csv(b, origin, h, v, ok)
    assert a.read_bytes() == b.read_bytes()
    w = v + np.random.default_rng(2).normal(size=v.shape)
    c = tmp_path / "c.csv"
    O.ref_grid_save_csv(c, origin, h, w, ok)
    ref = O.ref_grid_load_rmse(a, c)
    assert B.grid_rmse(v, w, ok, ok) == pytest.approx(ref, rel=1e-15)


def test_grid_csv_errors(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("x,y,v\n")
    with pytest.raises(B.ParseError):
        B.load_grid_csv(bad)
    bad.write_text("x,y,value,valid\n0,0,1\n")
    with pytest.raises(B.ParseError):
        B.load_grid_csv(bad)
    bad.write_text("x,y,value,valid\n0,0,1,1\n0.5,0,1,1\n2,0,1,1\n")  # irregular lattice
    with pytest.raises(B.ParseError):
        B.load_grid_csv(bad)
    with pytest.raises(B.ParseError):
        B.load_grid_csv(tmp_path / "missing.csv")
    with pytest.raises(B.ParseError):
        B.grid_rmse([1.0, 2.0], [1.0, 2.0], [0, 0], [1, 1])  # no jointly valid nodes


def test_grid_pgm(tmp_path):
    v = np.array([[0.0, 1.0, 2.0], [3.0, 4.0, 5.0]])
    ok = np.array([[1, 1, 1], [1, 0, 1]], bool)
    p = tmp_path / "g.pgm"
    B.save_grid_pgm(p, v, ok)
    data = p.read_bytes()
    header = b"P5\n3 2\n255\n"
    assert data.startswith(header)
    px = np.frombuffer(data[len(header):], np.uint8).reshape(2, 3)
    # top image row is the largest y; invalid pixels are black; linear map of [0, 5]
    assert px.tolist() == [[153, 0, 255], [0, 51, 102]]
    legend = (tmp_path / "g.pgm.txt").read_text()
    assert legend.startswith("min 0\nmax 5\n")


def test_streamline_csv_layout(tmp_path):
    seeds = np.array([[0.1, 0.2], [5.0, 5.0]])
    steps = 3
    pts = np.zeros((2, steps + 1, 2))
    pts[0, :3] = [[0.1, 0.2], [0.2, 0.2], [0.3, 0.2]]
    traced = dict(seeds=seeds, steps=steps, points=pts, counts=np.array([3, 0], np.int32),
                  reason_codes=np.array([1, 1], np.int32))
    p = tmp_path / "s.csv"
    B.write_streamlines_csv(p, traced)
    assert p.read_text().splitlines() == [
        "seed,step,x,y,reason", "0,0,0.10000000000000001,0.20000000000000001,",
        "0,1,0.20000000000000001,0.20000000000000001,", "0,2,0.29999999999999999,0.20000000000000001,",
        "0,-1,0.29999999999999999,0.20000000000000001,outside", "1,-1,5,5,outside"]
