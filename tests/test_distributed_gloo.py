"""World-size-2 CPU (gloo) tests of the multi-GPU host logic: M-sharded forward needs no
collective, and data-parallel gradients all-reduced through GradBucket / allreduce_grads equal
the full-batch gradients. The per-rank compute is the CPU oracle (test infrastructure)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_12211_b200.distributed import GradBucket, allreduce_grads, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(M=32, K=16, N=24, t=4, r=12):
    from oracle import stl_oracle as O
    rng = O.make_rng(5)
    e_x, e_w, d = O.random_gaussian_init(t, r, rng, scale=0.4)
    w = O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, t)
    x = rng.standard_normal((M, K))
    gy = rng.standard_normal((M, N))
    return t, r, e_x, d, w, x, gy


def _worker(rank, world, port, q):
    from oracle import stl_oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t, r, e_x, d, w, x, gy = _problem()
        lo, hi = shard_rows(x.shape[0], t, world, rank)
        y, cache = O.layer_forward_cached(x[lo:hi], w, e_x, d, t)
        g_ex, g_d, g_w, g_x = O.layer_backward(w, e_x, d, cache, gy[lo:hi], t)
        bucket = GradBucket(r, t, w.shape[1], w.shape[0], "cpu")
        bucket.g_w.copy_(torch.from_numpy(g_w.transpose(2, 1, 0).copy()))
        bucket.g_ex.copy_(torch.from_numpy(g_ex))
        bucket.g_d.copy_(torch.from_numpy(g_d))
        bucket.allreduce()
        a_ex, a_d = torch.from_numpy(g_ex.copy()), torch.from_numpy(g_d.copy())
        allreduce_grads([a_ex, a_d])
        q.put((rank, lo, hi, y, g_x, bucket.g_w.numpy().copy(), bucket.g_ex.numpy().copy(),
               bucket.g_d.numpy().copy(), a_ex.numpy(), a_d.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_rows_partition():
    for M, t, world in ((8192, 4, 8), (36, 4, 2), (12, 4, 4), (4, 4, 3)):
        cuts = [shard_rows(M, t, world, k) for k in range(world)]
        assert cuts[0][0] == 0 and cuts[-1][1] == M
        for (a, b), (c, _) in zip(cuts, cuts[1:]):
            assert b == c
        assert all(lo % t == 0 and hi % t == 0 for lo, hi in cuts)
    assert shard_rows(8192, 4, 8, 3, align=128) == (3072, 4096)
    with pytest.raises(ValueError):
        shard_rows(10, 4, 2, 0)


def test_dp_allreduce_world2_gloo():
    from oracle import stl_oracle as O
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    t, r, e_x, d, w, x, gy = _problem()
    y_full, cache = O.layer_forward_cached(x, w, e_x, d, t)
    g_ex, g_d, g_w, g_x = O.layer_backward(w, e_x, d, cache, gy, t)
    # forward: concatenated row slabs == full forward (no collective needed)
    y_cat = np.concatenate([res[3] for res in results])
    np.testing.assert_allclose(y_cat, y_full, atol=1e-12)
    np.testing.assert_allclose(np.concatenate([res[4] for res in results]), g_x, atol=1e-12)
    for res in results:  # every rank holds the full-batch gradients after the all-reduce
        np.testing.assert_allclose(res[5], g_w.transpose(2, 1, 0), rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(res[6], g_ex, rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(res[7], g_d, rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(res[8], g_ex, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(res[9], g_d, rtol=1e-12, atol=1e-12)
