"""The multi-rank STL path with the CUDA library on every rank (world size 2, gloo, both ranks
on the one GPU a test box has): the M-sharded forward (no collective) and the
data-parallel gradient all-reduce, checked against the single-process result."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

T, R, M, K, N = 4, 24, 2048, 512, 1024


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    import paper_2503_12211_b200 as stl

    dev = torch.device("cuda", 0)
    snf = stl.random_gaussian_init(T, R, stl.make_rng(0), scale=0.5).to(dev)
    g = torch.Generator(device=dev).manual_seed(0)
    w = (torch.randn((R, N // T, K // T), device=dev, generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
    gy = torch.randn((M, N), device=dev, generator=g).to(torch.bfloat16)
    return stl, snf, w, x, gy


def _worker(rank: int, world: int, port: int, out_dir: str) -> None:
    import torch.distributed as dist

    from paper_2503_12211_b200.distributed import GradBucket, shard_rows
    from paper_2503_12211_b200.layer import LayerCache, backward_raw
    from paper_2503_12211_b200.snf_operator import _forward

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    stl, snf, w, x, gy = _problem()
    # forward: this rank's token rows (multiple of 256 tiles), no collective
    lo, hi = shard_rows(M, T, world, rank, align=256)
    y = _forward(x[lo:hi].contiguous(), w, snf)
    parts = [torch.empty((M // world, N), dtype=torch.float32) for _ in range(world)]
    dist.all_gather(parts, y.float().cpu())
    # data parallel: this rank's batch = its row shard; all-reduce the bucketed gradients
    yk, u, ye = _forward(x[lo:hi].contiguous(), w, snf, keep_cache=True)
    g_ex, g_d, g_w, _ = backward_raw(snf, w, LayerCache(x[lo:hi].contiguous(), u, ye),
                                     gy[lo:hi].contiguous())
    bucket = GradBucket(R, T, N // T, K // T, "cpu")
    bucket.g_w.copy_(g_w.cpu())
    bucket.g_ex.copy_(g_ex.cpu())
    bucket.g_d.copy_(g_d.cpu())
    bucket.allreduce()
    if rank == 0:
        np.save(os.path.join(out_dir, "y_sharded.npy"), torch.cat(parts).numpy())
        np.save(os.path.join(out_dir, "grads_dp.npy"), bucket.flat.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_forward_and_dp_allreduce_with_cuda_ranks(tmp_path):
    import torch.multiprocessing as mp

    from paper_2503_12211_b200.layer import LayerCache, backward_raw
    from paper_2503_12211_b200.snf_operator import _forward

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    stl, snf, w, x, gy = _problem()
    y_full = _forward(x, w, snf).float().cpu().numpy()
    # rows of Y depend only on the same rows of X: the sharded forward is bit-identical
    assert np.array_equal(np.load(tmp_path / "y_sharded.npy"), y_full)
    # DP gradients = gradients of the whole batch (sums over token rows), fp32 reorder only
    yk, u, ye = _forward(x, w, snf, keep_cache=True)
    g_ex, g_d, g_w, _ = backward_raw(snf, w, LayerCache(x, u, ye), gy)
    want = torch.cat([g_w.reshape(-1), g_ex.reshape(-1), g_d.reshape(-1)]).cpu().numpy()
    got = np.load(tmp_path / "grads_dp.npy")
    assert np.linalg.norm(got - want) <= 1e-5 * np.linalg.norm(want)
