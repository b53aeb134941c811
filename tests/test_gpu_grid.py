"""GPU PhotonGrid parity: keys, permutation, cell ranges and query_ball order
(photon_map.cpp:26-78; reference tests test_photon_map.cpp)."""
import numpy as np
import pytest

from paper_2504_04411_b200 import InvalidArgument, PhotonGrid

pytestmark = pytest.mark.gpu


def _rand_pos(rng, n, extent):
    return (extent * (2 * rng.random((n, 3)) - 1)).astype(np.float32)


@pytest.mark.parametrize("n,extent,cell", [(2500, 2.0, 0.3), (100000, 1.0, 0.05), (7, 1.0, 0.5)])
def test_grid_internals_match(port, n, extent, cell):
    rng = np.random.default_rng(n)
    pos = _rand_pos(rng, n, extent)
    g = PhotonGrid(pos, cell)
    keys, b, e, order = g.internals()
    og = port.grid_build(pos.astype(np.float64), cell)
    k2, b2, e2, o2 = og.export()
    assert np.array_equal(keys, k2)
    assert np.array_equal(b, b2) and np.array_equal(e, e2)
    assert np.array_equal(order, o2)


def test_query_ball_matches_in_order(port):
    rng = np.random.default_rng(31)
    cell = 0.3
    pos = _rand_pos(rng, 2500, 2.0)
    g = PhotonGrid(pos, cell)
    og = port.grid_build(pos.astype(np.float64), cell)
    centers = 2.4 * (2 * rng.random((200, 3)) - 1)
    radii = cell * (0.3 + 0.7 * rng.random(200))
    radii[:10] = cell  # r == cell is allowed (test_photon_map.cpp:62-74)
    got = g.query_ball_batch(centers, radii)
    nonempty = 0
    for q in range(200):
        want = og.query_ball(centers[q], radii[q])
        assert np.array_equal(got[q], want)
        nonempty += len(want) > 0
    assert nonempty > 50


def test_empty_grid_and_errors():
    g = PhotonGrid(np.zeros((0, 3)), 0.5)
    assert g.size() == 0
    assert len(g.query_ball([0, 0, 0], 0.25)) == 0
    assert len(g.query_ball([0, 0, 0], 5.0)) == 0  # empty grid returns before the r check
    with pytest.raises(InvalidArgument):
        PhotonGrid(np.zeros((0, 3)), 0.0)
    with pytest.raises(InvalidArgument):
        PhotonGrid(np.zeros((0, 3)), -1.0)
    g1 = PhotonGrid(np.zeros((1, 3)), 0.5)
    with pytest.raises(InvalidArgument):
        g1.query_ball([0, 0, 0], 0.5001)


def test_closed_ball_and_insertion_order():
    vs = np.array([[0.5, 0, 0], [0, 0.5, 0], [0.5001, 0, 0]], np.float32)
    g = PhotonGrid(vs, 0.5)
    found = sorted(g.query_ball([0, 0, 0], 0.5).tolist())
    assert found == [0, 1]
    vs = np.array([[0.01 * i, 0, 0] for i in range(10)], np.float32)
    g = PhotonGrid(vs, 1.0)
    assert g.query_ball([0.05, 0, 0], 0.5).tolist() == list(range(10))


def test_rebuild_deterministic():
    rng = np.random.default_rng(33)
    pos = _rand_pos(rng, 800, 1.5)
    a, b = PhotonGrid(pos, 0.2), PhotonGrid(pos, 0.2)
    c = 1.5 * (2 * rng.random((100, 3)) - 1)
    r = 0.2 * rng.random(100)
    for x, y in zip(a.query_ball_batch(c, r), b.query_ball_batch(c, r)):
        assert np.array_equal(x, y)
