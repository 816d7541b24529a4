"""GPU parity of the 4-NN point-size initialisation (trips_knn_sizes) against the oracle's brute
force: bit-exact neighbour indices and sizes (same pinned fp32 sequence)."""
import numpy as np
import pytest
import torch

from oracle import oracle
from synth import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def run(pos, dev):
    from paper_2401_06003_b200 import knn_sizes
    s, nb = knn_sizes(torch.from_numpy(np.ascontiguousarray(pos, np.float32)).to(dev), return_neighbors=True)
    torch.cuda.synchronize()
    return s.cpu().numpy(), nb.cpu().numpy()


@pytest.mark.parametrize("seed", range(4))
def test_random_clouds_exact(dev, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 6000))
    p = (rng.normal(size=(n, 3)) * rng.uniform(0.1, 5, 3)).astype(np.float32)
    s, nb = run(p, dev)
    so, nbo = oracle.knn4(p)
    assert np.array_equal(nb, nbo)
    assert np.array_equal(s.view(np.uint32), so.view(np.uint32))


def test_structured_and_degenerate(dev):
    g = np.stack(np.meshgrid(np.arange(12), np.arange(9), np.arange(7), indexing="ij"), -1).reshape(-1, 3)
    p = g.astype(np.float32) * np.float32(0.5)                 # exact ties everywhere
    p = np.concatenate([p, p[:10], [[np.nan, 0, 0], [np.inf, 1, 1]], np.zeros((1, 3))]).astype(np.float32)
    s, nb = run(p, dev)
    so, nbo = oracle.knn4(p)
    assert np.array_equal(nb, nbo) and np.array_equal(s.view(np.uint32), so.view(np.uint32))
    for q in ([[0, 0, 0]], [[0, 0, 0], [1, 1, 1]], np.zeros((5, 3))):
        q = np.asarray(q, np.float32)
        s, nb = run(q, dev)
        so, nbo = oracle.knn4(q)
        assert np.array_equal(nb, nbo) and np.array_equal(s, so)


def test_surface_cloud_sampled(dev):
    """A C2-like surface cloud (planar patches: most grid cells empty), 1M points, checked on
    sampled query points against the brute force over all points."""
    sc = scenes.make_config("C2", n=1_000_000)
    s, nb = run(sc.pos, dev)
    q = np.random.default_rng(1).choice(sc.n, 300, replace=False)
    so, nbo = oracle.knn4(sc.pos, queries=q)
    assert np.array_equal(nb[q], nbo)
    assert np.array_equal(s[q].view(np.uint32), so.view(np.uint32))
    assert s.min() >= 0 and np.isfinite(s).all()


def test_clusters_duplicates_and_wide_extent(dev):
    """Morton-window edge cases: dense clusters far apart (octree boundaries between a point and
    its neighbours), 3000 copies of one point (ties broken by index), a huge-extent outlier pair,
    and tiny clouds where the window covers everything."""
    rng = np.random.default_rng(5)
    cl = [rng.normal(size=(800, 3)) * 1e-3 + rng.uniform(-10, 10, 3) for _ in range(6)]
    dup = np.repeat(np.array([[0.25, -0.5, 3.0]]), 3000, 0)
    wide = np.array([[1e30, 0, 0], [-1e30, 5, 5], [1e30, 1, 0]])
    p = np.concatenate(cl + [dup, wide]).astype(np.float32)
    p = p[rng.permutation(len(p))]
    s, nb = run(p, dev)
    so, nbo = oracle.knn4(p)
    assert np.array_equal(nb, nbo) and np.array_equal(s.view(np.uint32), so.view(np.uint32))
    for n in (2, 3, 5, 9, 17, 18, 40):
        q = rng.normal(size=(n, 3)).astype(np.float32)
        s, nb = run(q, dev)
        so, nbo = oracle.knn4(q)
        assert np.array_equal(nb, nbo) and np.array_equal(s.view(np.uint32), so.view(np.uint32))


def test_c4_cloud_full_size_sampled(dev):
    """The bench's kNN workload: the 8M-point C4 cloud, sampled queries against the brute force."""
    sc = scenes.make_config("C4", n_views=1)
    s, nb = run(sc.pos, dev)
    q = np.random.default_rng(2).choice(sc.n, 200, replace=False)
    so, nbo = oracle.knn4(sc.pos, queries=q)
    assert np.array_equal(nb[q], nbo)
    assert np.array_equal(s[q].view(np.uint32), so.view(np.uint32))
    assert s.min() >= 0 and np.isfinite(s).all()
