"""Multi-process (world_size 2, gloo, CPU) tests of the view-parallel step the GPU bench runs:
dist.batch_step with its reductions (all-reduce, reduce-scatter into padded shards, asynchronous
issue) and dist.PipelinedSteps' double-buffered overlap.  The per-view renderer here is the CPU
oracle writing the library's flat gradient layout [pos_size 4n | desc F n | opacity n | pad];
on GPUs dist.CudaViewRenderer plugs into the same batch_step (bench.py, the GPU parity tests).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_06003_b200 import dist as tdist

N_VIEWS = 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from synth import scenes
    sc = scenes.make_config("C4", n=2001, n_views=N_VIEWS)      # odd n: the flat buffer needs padding
    cams = [scenes.look_at(-c.R.T.astype(np.float64) @ c.t.astype(np.float64), [0, 0, 0], 48, 32, 30.0)
            for c in sc.cams]
    return sc, cams


def _flat(g, n, F):
    """oracle rows [n, 5+F] (pos, s_w, alpha, tau) -> the library's flat layout (unpadded)."""
    return np.concatenate([g[:, 0:4].reshape(-1), g[:, 5:5 + F].reshape(-1), g[:, 4]])


class _OracleRenderer:
    """render_view with begin/end hooks like dist.CudaViewRenderer; accumulates the oracle's
    gradients of view v (upstream gradient seeded by v) into the flat buffer."""

    def __init__(self, sc, cams):
        from oracle import oracle
        self.sc, self.cams = sc, cams
        self.P = oracle.num_pixels(48, 32, 4)
        self.calls = []

    def begin(self):
        self.calls.append("begin")

    def __call__(self, v, grad):
        from oracle import oracle
        from synth import scenes
        sc = self.sc
        G = scenes.grad_pyramid(self.P * (sc.F + 1), seed=v)
        g, _ = oracle.backward(self.cams[v], 4, sc.pos, sc.sw, sc.alpha, sc.desc, G)
        f = _flat(g, sc.n, sc.F)
        grad[:f.size] += torch.from_numpy(f)
        self.calls.append(v)

    def end(self):
        self.calls.append("end")


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc, cams = _scene()
    views = tdist.shard_views(N_VIEWS, rank, world)
    nf = tdist.padded_numel((5 + sc.F) * sc.n, world)
    # 1. synchronous all-reduce (every rank holds the sum)
    r = _OracleRenderer(sc, cams)
    grad = torch.full((nf,), 3.0, dtype=torch.float64)            # zeroed by the step
    assert tdist.batch_step(r, views, grad, world=world) is None
    assert r.calls[0] == "begin" and r.calls[-1] == "end" and r.calls[1:-1] == views
    np.save(os.path.join(out_dir, f"ar{rank}.npy"), grad.numpy())
    # 2. asynchronous reduce-scatter into this rank's shard
    shard = torch.empty(nf // world, dtype=torch.float64)
    g2 = torch.zeros(nf, dtype=torch.float64)
    h = tdist.batch_step(_OracleRenderer(sc, cams), views, g2, world=world, reduce="reduce_scatter", out=shard,
                         async_op=True)
    h.wait()
    np.save(os.path.join(out_dir, f"rs{rank}.npy"), shard.numpy())
    # 3. pipelined steps: double-buffered gradients, step k's reduction in flight during step k+1
    grads = [torch.zeros(nf, dtype=torch.float64) for _ in range(2)]
    seen = []

    def step(g, k):
        seen.append((k, g.data_ptr()))
        return tdist.batch_step(_OracleRenderer(sc, cams), views, g, world=world, async_op=True)
    tdist.PipelinedSteps(grads).run(3, step)
    assert [p for _, p in seen] == [grads[0].data_ptr(), grads[1].data_ptr(), grads[0].data_ptr()]
    np.save(os.path.join(out_dir, f"pl{rank}.npy"), np.stack([g.numpy() for g in grads]))
    np.save(os.path.join(out_dir, f"v{rank}.npy"), np.array(views))
    dist.destroy_process_group()


def test_shard_helpers():
    for n in (1, 5, 32):
        for w in (1, 2, 3, 8):
            allv = sorted(v for r in range(w) for v in tdist.shard_views(n, r, w))
            assert allv == list(range(n))
    with pytest.raises(ValueError):
        tdist.shard_views(4, 2, 2)
    for numel in (1, 9 * 2001, 9 * 8_000_000):
        for w in (1, 2, 3, 8):
            p = tdist.padded_numel(numel, w)
            assert p >= numel and p % w == 0 and (p // w) % 4 == 0 and p - numel < 4 * w
            rngs = [tdist.shard_range(p, r, w) for r in range(w)]
            assert rngs[0][0] == 0 and rngs[-1][1] == p and all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))


def test_flat_inputs_layout():
    n, F = 7, 4
    pos = torch.arange(3 * n, dtype=torch.float32).view(n, 3)
    sw, al = torch.arange(n, dtype=torch.float32) + 100, torch.arange(n, dtype=torch.float32) + 200
    de = torch.arange(F * n, dtype=torch.float32).view(n, F) + 300
    flat, n2, F2 = tdist.flat_inputs(pos, sw, al, de, world=3)
    assert (n2, F2) == (n, F) and flat.numel() % 3 == 0 and flat.numel() >= (5 + F) * n
    p, s, a, d = tdist.input_views(flat, n, F)
    assert torch.equal(p, pos) and torch.equal(s, sw) and torch.equal(a, al) and torch.equal(d, de)


def test_view_parallel_reductions_gloo(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    v0, v1 = (np.load(tmp_path / f"v{r}.npy") for r in range(world))
    assert sorted(list(v0) + list(v1)) == list(range(N_VIEWS)) and not set(v0) & set(v1)
    sc, cams = _scene()
    nf = tdist.padded_numel((5 + sc.F) * sc.n, world)
    ref = torch.zeros(nf, dtype=torch.float64)
    rv = _OracleRenderer(sc, cams)
    for v in range(N_VIEWS):
        rv(v, ref)
    ref = ref.numpy()
    assert np.abs(ref).sum() > 0 and not ref[(5 + sc.F) * sc.n:].any()
    ar = [np.load(tmp_path / f"ar{r}.npy") for r in range(world)]
    assert np.array_equal(ar[0], ar[1])                                   # all-reduce: identical on ranks
    assert np.allclose(ar[0], ref, rtol=1e-12, atol=1e-12)
    rs = np.concatenate([np.load(tmp_path / f"rs{r}.npy") for r in range(world)])
    assert np.allclose(rs, ref, rtol=1e-12, atol=1e-12)                   # shards tile the sum
    for r in range(world):
        pl = np.load(tmp_path / f"pl{r}.npy")
        assert np.allclose(pl[0], ref, rtol=1e-12, atol=1e-12) and np.allclose(pl[1], ref, rtol=1e-12, atol=1e-12)
