"""T2T-ViT-7 with STL projections: the token plumbing of PAPER.md:581-583
and an STL token layer checked against a plain PyTorch fp32 restatement of the operator."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2503_12211_b200 import t2t_vit


def test_square_order_groups_2x2_patches():
    o = t2t_vit.square_order(14, 14)
    assert sorted(o.tolist()) == list(range(196))
    for k in range(49):
        quad = o[4 * k:4 * k + 4].tolist()
        rows, cols = {i // 14 for i in quad}, {i % 14 for i in quad}
        assert len(rows) == 2 and len(cols) == 2 and max(rows) - min(rows) == 1


def _ar_worker(rank, world, port, out):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    ps = [torch.nn.Parameter(torch.zeros(3, 2)), torch.nn.Parameter(torch.zeros(5))]
    for i, p in enumerate(ps):
        p.grad = torch.full_like(p, float(rank + 1) * (i + 1))
    t2t_vit.allreduce_grads(ps)
    out[rank] = [p.grad.clone() for p in ps]
    dist.destroy_process_group()


def test_allreduce_grads_gloo_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = mp.Manager().dict()
    mp.spawn(_ar_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        g0, g1 = out[r]
        assert torch.allclose(g0, torch.full((3, 2), 1.5)) and torch.allclose(g1, torch.full((5,), 3.0))


def _stl_torch_fp32(x, planes, e_x, d, t):
    """Plain fp32 PyTorch STL (reference semantics: encode, r slice GEMMs, decode)."""
    M, K = x.shape
    bi, bk = M // t, K // t
    tiles = x.reshape(bi, t, bk, t).permute(0, 2, 1, 3).reshape(bi, bk, t * t)
    u = torch.einsum("ijc,pc->pij", tiles, e_x)                    # (r, bi, bk)
    yenc = torch.bmm(u, planes.transpose(1, 2))                      # (r, bi, bj)
    ytile = torch.einsum("pij,pc->ijc", yenc, d)
    bj = ytile.shape[1]
    return ytile.reshape(bi, bj, t, t).permute(0, 2, 1, 3).reshape(M, bj * t)


@pytest.mark.gpu
def test_stl_token_linear_fold_matches_torch_fp32():
    torch.manual_seed(0)
    lay = t2t_vit.StlTokenLinear(256, 512, t=4, r=24, seed=3)
    x = torch.randn(3, 197, 256, device="cuda").to(torch.bfloat16).requires_grad_(True)
    y = lay(x)
    assert y.shape == (3, 197, 512)
    # fp32 restatement with the same (bf16-rounded) weights
    w = lay.w_planes.detach().to(torch.bfloat16).float().requires_grad_(True)
    e_x = lay.e_x.detach().clone().requires_grad_(True)
    d = lay.d.detach().clone().requires_grad_(True)
    xr = x.detach().float().requires_grad_(True)
    xp = torch.nn.functional.pad(xr, (0, 0, 0, 3))
    yr = _stl_torch_fp32(xp.reshape(600, 256), w, e_x, d, 4).reshape(3, 200, 512)
    yr = torch.cat([yr[:, :196], torch.einsum("btn,t->bn", yr[:, 196:], lay.fold.detach())[:, None]], 1)
    rel = (y.float() - yr).norm() / yr.norm()
    assert rel < 1e-2, rel
    gy = torch.randn_like(yr)
    (y.float() * gy).sum().backward()
    (yr * gy).sum().backward()
    for got, ref in ((x.grad.float(), xr.grad), (lay.e_x.grad, e_x.grad), (lay.d.grad, d.grad),
                     (lay.w_planes.grad, w.grad)):
        assert ((got - ref).norm() / ref.norm()) < 2e-2


@pytest.mark.gpu
def test_t2t_vit7_train_step():
    torch.manual_seed(0)
    model = t2t_vit.T2TViT7(num_classes=10, stl=True)
    n_stl = sum(isinstance(m, t2t_vit.StlTokenLinear) for m in model.modules())
    assert n_stl == 28                                             # qkv, proj, fc1, fc2 x 7
    opt = torch.optim.AdamW(model.parameters(), lr=1e-3)
    img = torch.randn(2, 3, 224, 224, device="cuda")
    labels = torch.tensor([1, 7], device="cuda")
    before = model.blocks[0].fc1.w_planes.detach().clone()
    losses = [float(t2t_vit.train_step(model, opt, img, labels)) for _ in range(3)]
    assert all(np.isfinite(losses)) and losses[-1] < losses[0]
    assert not torch.equal(before, model.blocks[0].fc1.w_planes.detach())


@pytest.mark.gpu
def test_token_kernels_match_framework_ops():
    """stl_token_pad / unpad / fold / fold_backward against the same plumbing in torch ops."""
    torch.manual_seed(1)
    dev = torch.device("cuda")
    B, T, C, N, t = 5, 197, 48, 64, 4
    Tp = T - 1 + t
    for dt in (torch.float32, torch.bfloat16):
        x = torch.randn(B, T, C, device=dev, dtype=dt, requires_grad=True)
        xp = t2t_vit.TokenPad.apply(x, Tp, 56)
        ref = torch.nn.functional.pad(x.detach().to(torch.bfloat16), (0, 8, 0, Tp - T))
        assert torch.equal(xp, ref)
        g = torch.randn(B, Tp, 56, device=dev).to(torch.bfloat16)
        xp.backward(g)
        assert x.grad.dtype == dt and torch.equal(x.grad, g[:, :T, :C].to(dt))
    y = torch.randn(B, Tp, N, device=dev).to(torch.bfloat16).requires_grad_(True)
    fold = torch.randn(t, device=dev, requires_grad=True)
    bias = torch.randn(N, device=dev, requires_grad=True)
    out = t2t_vit.TokenFold.apply(y, fold, bias, T)
    yr = y.detach().float().requires_grad_(True)
    fr = fold.detach().clone().requires_grad_(True)
    br = bias.detach().clone().requires_grad_(True)
    last = torch.einsum("btn,t->bn", yr[:, T - 1:], fr)
    ref = torch.cat([yr[:, :T - 1], last[:, None]], 1) + br
    assert out.shape == (B, T, N)
    assert ((out.float() - ref).abs() <= 1e-2 * ref.abs() + 1e-3).all()
    go = torch.randn(B, T, N, device=dev).to(torch.bfloat16)
    out.backward(go)
    ref.backward(go.float())
    assert ((y.grad.float() - yr.grad).abs() <= 1e-2 * yr.grad.abs() + 1e-3).all()
    assert torch.allclose(fold.grad, fr.grad, rtol=1e-4, atol=1e-3)
    assert torch.allclose(bias.grad, br.grad, rtol=1e-4, atol=1e-3)


@pytest.mark.gpu
def test_stl_token_linear_fused_plumbing_matches_framework_ops():
    torch.manual_seed(2)
    lay = t2t_vit.StlTokenLinear(256, 512, t=4, r=24, seed=5)
    with torch.no_grad():
        lay.fold.copy_(torch.tensor([0.7, 0.2, -0.4, 0.3]))
        lay.bias.normal_()
    x0 = torch.randn(4, 197, 256, device="cuda")
    gy = torch.randn(4, 197, 512, device="cuda").to(torch.bfloat16)
    res = {}
    for fused in (True, False):
        t2t_vit.FUSED_TOKEN_PLUMBING = fused
        try:
            lay.zero_grad(set_to_none=True)
            x = x0.clone().requires_grad_(True)
            y = lay(x)
            y.backward(gy)
            res[fused] = [y.float(), x.grad, lay.fold.grad, lay.bias.grad, lay.e_x.grad,
                          lay.d.grad, lay.w_planes.grad]
        finally:
            t2t_vit.FUSED_TOKEN_PLUMBING = True
    for a, b in zip(res[True], res[False]):
        assert ((a - b).norm() / b.norm()) < 5e-3
