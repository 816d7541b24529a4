"""The comparator networks compiled into k_raster (csrc/kernels.cuh) sort every input and the
merge keeps exactly the 16 smallest keys: checked exhaustively with the 0-1 principle
(a comparator network sorts all inputs iff it sorts all 0/1 inputs)."""
import itertools
import os
import re

import numpy as np

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2401_06003_b200",
                   "csrc", "kernels.cuh")


def network(n, branch=0):
    """Comparators of sort_small<n> as compiled; for a body with an #if/#else (TRIPS_NET16),
    branch 0 is the default (#if) network and branch 1 the #else one."""
    src = open(SRC).read()
    body = src.split(f"sort_small<{n}>(uint64_t (&t)[16])\n{{", 1)[1].split("\n}", 1)[0]
    if "#else" in body:
        body = body.split("#else")[branch]
    return [(int(a), int(b)) for a, b in re.findall(r"cswap\(t\[(\d+)\], t\[(\d+)\]\)", body)]


def apply(net, a):
    a = np.array(a)
    for i, j in net:
        lo, hi = np.minimum(a[..., i], a[..., j]), np.maximum(a[..., i], a[..., j])
        a[..., i], a[..., j] = lo, hi
    return a


def all_binary(n):
    return ((np.arange(1 << n)[:, None] >> np.arange(n)) & 1).astype(np.int8)


def _sorts_all(net, n):
    out = apply(net, all_binary(n))
    return bool(np.all(np.diff(out, axis=1) >= 0))


def test_sort4_network_sorts():
    net = network(4)
    assert len(net) == 5 and all(i < j < 4 for i, j in net)
    assert _sorts_all(net, 4)


def test_sort8_network_sorts():
    net = network(8)
    assert len(net) == 19 and all(i < j < 8 for i, j in net)
    assert _sorts_all(net, 8)


def test_sort12_network_sorts():
    net = network(12)
    assert len(net) == 39 and all(i < j < 12 for i, j in net)
    assert _sorts_all(net, 12)


def test_sort16_network_sorts():
    net = network(16)                    # default: 60 comparators
    assert len(net) == 60 and all(i < j < 16 for i, j in net)
    assert _sorts_all(net, 16)
    batcher = network(16, branch=1)      # TRIPS_NET16 = 0
    assert len(batcher) == 63 and all(i < j < 16 for i, j in batcher)
    assert _sorts_all(batcher, 16)


def test_networks_fail_when_a_comparator_is_dropped():
    """The exhaustive check has teeth: every comparator of the 12- and 16-key networks is needed."""
    for n in (12, 16):
        net = network(n)
        for k in range(len(net)):
            assert not _sorts_all(net[:k] + net[k + 1:], n)


def merge_keep16(r, t, n):
    """Python restatement of merge_keep16<N>: r, t sorted ascending, t valid in t[0:n]."""
    r = np.array(r)
    for j in range(16 - n, 16):
        r[..., j] = np.minimum(r[..., j], t[..., 15 - j])
    for d in (8, 4, 2, 1):
        for i in range(16):
            if i & d == 0:
                lo, hi = np.minimum(r[..., i], r[..., i + d]), np.maximum(r[..., i], r[..., i + d])
                r[..., i], r[..., i + d] = lo, hi
    return r


def test_merge_keeps_16_smallest_random():
    """Random distinct keys (the kernel's keys are unique): merge = sort(union)[:16]."""
    rng = np.random.default_rng(0)
    for n in (4, 8, 12, 16):
        for _ in range(3000):
            keys = rng.permutation(1000)[:16 + n]
            r = np.sort(keys[:16])
            t = np.full(16, 10 ** 9)
            t[:n] = np.sort(keys[16:])
            got = merge_keep16(r[None], t[None], n)[0]
            assert np.array_equal(got, np.sort(keys)[:16])


def test_merge_zero_one_exhaustive_small():
    """0-1 principle on the merge for all sorted 0/1 inputs (r and t sorted: 17 x 17 cases)."""
    for n in (4, 8, 12, 16):
        for a, b in itertools.product(range(17), range(n + 1)):
            r = np.array([0] * a + [1] * (16 - a))
            t = np.array([0] * b + [1] * (16 - b))
            t[n:] = 1
            got = merge_keep16(r[None], t[None], n)[0]
            zeros = min(16, a + b)
            assert np.array_equal(got, np.array([0] * zeros + [1] * (16 - zeros)))
