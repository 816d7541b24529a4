"""Multi-process (world_size 2, gloo, CPU) test of the view-parallel step: views are sharded
without overlap and the all-reduced gradient equals the single-process sum over all views.
The per-view renderer here is the CPU oracle (the CUDA renderer plugs into the same
batch_step on GPUs); this covers the host-side sharding and reduction logic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_06003_b200 import dist as tdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from synth import scenes
    sc = scenes.make_config("C4", n=2000, n_views=5)
    cams = [scenes.look_at(-c.R.T.astype(np.float64) @ c.t.astype(np.float64), [0, 0, 0], 48, 32, 30.0)
            for c in sc.cams]
    return sc, cams


def _oracle_renderer(sc, cams):
    from oracle import oracle
    from synth import scenes
    P = oracle.num_pixels(48, 32, 4)

    def render_view(v, grad):
        G = scenes.grad_pyramid(P * 5, seed=v)
        g, _ = oracle.backward(cams[v], 4, sc.pos, sc.sw, sc.alpha, sc.desc, G)
        grad += torch.from_numpy(g)
    return render_view


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc, cams = _scene()
    views = tdist.shard_views(len(cams), rank, world)
    grad = torch.zeros(sc.n, 5 + sc.F, dtype=torch.float64)
    tdist.batch_step(_oracle_renderer(sc, cams), views, grad, world=world)
    np.save(os.path.join(out_dir, f"g{rank}.npy"), grad.numpy())
    np.save(os.path.join(out_dir, f"v{rank}.npy"), np.array(views))
    dist.destroy_process_group()


def test_shard_views_partition():
    for n in (1, 5, 32):
        for w in (1, 2, 3, 8):
            allv = sorted(v for r in range(w) for v in tdist.shard_views(n, r, w))
            assert allv == list(range(n))
    with pytest.raises(ValueError):
        tdist.shard_views(4, 2, 2)


def test_view_parallel_allreduce_gloo(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g0, g1 = (np.load(tmp_path / f"g{r}.npy") for r in range(world))
    v0, v1 = (np.load(tmp_path / f"v{r}.npy") for r in range(world))
    assert sorted(list(v0) + list(v1)) == list(range(5)) and not set(v0) & set(v1)
    assert np.array_equal(g0, g1)                                   # all-reduce: identical on ranks
    sc, cams = _scene()
    ref = torch.zeros(sc.n, 5 + sc.F, dtype=torch.float64)
    rv = _oracle_renderer(sc, cams)
    for v in range(len(cams)):
        rv(v, ref)
    assert np.allclose(g0, ref.numpy(), rtol=1e-12, atol=1e-12)
    assert np.abs(ref.numpy()).sum() > 0
