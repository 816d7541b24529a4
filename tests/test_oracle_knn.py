"""Pins of the oracle's 4-nearest-neighbour size initialisation (SURVEY.md 8(f)
row 4): SPEC.md:117-119 examples, a library k-d tree (scipy cKDTree, fp64) on random clouds,
and degenerate inputs."""
import numpy as np
import pytest

from oracle import oracle


def test_spec_examples():
    # two points at distance 1 -> both sizes 1
    s, nb = oracle.knn4(np.array([[0, 0, 0], [1, 0, 0]], np.float32))
    assert list(s) == [1.0, 1.0] and list(nb[0]) == [1, -1, -1, -1] and list(nb[1]) == [0, -1, -1, -1]
    # unit-spacing 3-D grid, interior point -> 4 nearest at distance 1
    g = np.stack(np.meshgrid(np.arange(5), np.arange(5), np.arange(5), indexing="ij"), -1).reshape(-1, 3)
    s, nb = oracle.knn4(g.astype(np.float32))
    interior = np.all((g > 0) & (g < 4), axis=1)
    assert np.all(s[interior] == 1.0)
    # ties at equal distance break on the neighbour index
    i = int(np.nonzero((g == [2, 2, 2]).all(1))[0][0])
    six = sorted(int(j) for j in np.nonzero(np.abs(g - g[i]).sum(1) == 1)[0])
    assert list(nb[i]) == six[:4]


@pytest.mark.parametrize("seed", range(3))
def test_matches_kdtree(seed):
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    p = rng.normal(size=(3000, 3)).astype(np.float32) * rng.uniform(0.5, 3, 3).astype(np.float32)
    s, nb = oracle.knn4(p)
    d, j = cKDTree(p.astype(np.float64)).query(p.astype(np.float64), k=6)
    # exclude self (first column); compare the 4 nearest where the 4th/5th are well separated
    sep = d[:, 5] - d[:, 4] > 1e-5 * d[:, 4]
    assert sep.mean() > 0.99
    assert np.array_equal(np.sort(nb[sep], 1), np.sort(j[sep, 1:5], 1))
    ref = d[:, 1:5].mean(1)
    assert np.all(np.abs(s - ref) <= 1e-5 * ref)


def test_degenerate_inputs():
    s, nb = oracle.knn4(np.zeros((1, 3), np.float32))
    assert s[0] == 0 and list(nb[0]) == [-1] * 4
    p = np.array([[0, 0, 0], [0, 0, 0], [np.nan, 0, 0], [3, 0, 0]], np.float32)
    s, nb = oracle.knn4(p)
    assert list(nb[0][:3]) == [1, 3, -1]            # duplicate at distance 0 counts; NaN excluded
    assert s[0] == np.float32(3.0) / np.float32(2.0) and s[2] == 0
