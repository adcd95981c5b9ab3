"""T2T-ViT-7 with STL projections (BASELINE configs[3], configs[4]).

The model of the paper's Class-1 experiment: T2T-ViT-7
(Yuan et al., ICCV 2021; not part of /root/reference) with the activation x weight
linear layers replaced by STL layers of tile size t and rank r:

* trunk (7 blocks, embed 256, 4 heads, MLP 512): qkv, attention projection, fc1, fc2 — the
  paper's main replacement (79% of the FLOPs);
* optionally the T2T module's linear layers too (``stl_t2t=True``, the paper's follow-up), with
  input features zero-padded to a multiple of 8 t where the width is not tileable (147 -> 160).

STL-specific plumbing, as the paper describes it:

* 197 tokens are not divisible by t = 4: each STL layer appends 3 null token rows per sample
  (197 -> 200) and folds the last 4 output rows back into one row with 4 learnable coefficients
  (initialised (1, 0, 0, 0)); the summary (class) token sits at position 196, after the patches,
  so that fold acts on it;
* the 14 x 14 patch tokens are reordered once so that every 2 x 2 square of patches is 4
  consecutive tokens (one STL tile row group), instead of raster order.

Parameters are fp32 masters; activations run in bf16 (STL layers through the C ABI, the rest —
LayerNorm, softmax attention, the T2T performer, unfold — as plain PyTorch ops, which are not
the hot path). DP training: ``train_step`` all-reduces gradients over NCCL when a process group
is initialised (bench_t2t.py / scripts).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.nn as nn
import torch.nn.functional as F

from . import _lib
from .layer import StlLinearFunction
from .snf_operator import _stream, encode_tiles, weights_to_planes
from .strassen_basis import pruned_subset_init, random_gaussian_init, strassen_rank49


def make_triple(t: int, r: int, init: str, seed: int):
    rng = np.random.Generator(np.random.PCG64(seed))
    if init == "strassen" and t == 4:
        full = strassen_rank49()
        return full if r == 49 else pruned_subset_init(full, r, rng)
    return random_gaussian_init(t, r, rng, scale=0.5)


# The one-pass token plumbing kernels (TokenPad / TokenFold) are used whenever they apply;
# False routes through the framework-op version (A/B tests).
FUSED_TOKEN_PLUMBING = True


def _dt(dtype: torch.dtype) -> int:
    return _lib.STL_BF16 if dtype == torch.bfloat16 else _lib.STL_F32


class TokenPad(torch.autograd.Function):
    """(B, T, C) fp32/bf16 -> bf16 (B, Tp, Cp) with zero rows / columns in one pass
    (stl_token_pad); backward = stl_token_unpad into the input's dtype."""

    @staticmethod
    def forward(ctx, x, Tp: int, Cp: int):
        x = x.contiguous()
        B, T, C = x.shape
        out = torch.empty((B, Tp, Cp), dtype=torch.bfloat16, device=x.device)
        _lib.check(_lib.load().stl_token_pad(x.data_ptr(), _dt(x.dtype), B, T, C, out.data_ptr(),
                                             Tp, Cp, _stream(x.device)))
        ctx.shape, ctx.dtype = (B, T, C), x.dtype
        return out

    @staticmethod
    def backward(ctx, g):
        B, T, C = ctx.shape
        g = g.to(torch.bfloat16).contiguous()
        Tp, Cp = g.shape[1], g.shape[2]
        out = torch.empty((B, T, C), dtype=ctx.dtype, device=g.device)
        _lib.check(_lib.load().stl_token_unpad(g.data_ptr(), B, Tp, Cp, out.data_ptr(),
                                               _dt(ctx.dtype), T, C, _stream(g.device)))
        return out, None, None


class TokenFold(torch.autograd.Function):
    """(B, Tp, N) bf16 -> (B, T, N): the last t rows of each sample folded into one with the t
    learnable coefficients, + bias, in one pass (stl_token_fold); the backward writes d y and
    the fixed-order d bias / d fold sums in one pass plus a tree reduction."""

    @staticmethod
    def forward(ctx, y, fold, bias, T: int):
        y = y.contiguous()
        B, Tp, N = y.shape
        t = fold.numel()
        fold32 = fold.detach().float().contiguous()
        b32 = bias.detach().float().contiguous() if bias is not None else None
        out = torch.empty((B, T, N), dtype=torch.bfloat16, device=y.device)
        _lib.check(_lib.load().stl_token_fold(y.data_ptr(), B, Tp, N, t, fold32.data_ptr(),
                                              b32.data_ptr() if b32 is not None else None,
                                              out.data_ptr(), T, _stream(y.device)))
        ctx.save_for_backward(y, fold32)
        ctx.T, ctx.has_bias = T, bias is not None
        return out

    @staticmethod
    def backward(ctx, g):
        y, fold32 = ctx.saved_tensors
        B, Tp, N = y.shape
        t, T = fold32.numel(), ctx.T
        g = g.to(torch.bfloat16).contiguous()
        lib = _lib.load()
        gy = torch.empty_like(y)
        ws_n = int(lib.stl_token_fold_ws_floats(B, T, N, t))
        ws = torch.empty(ws_n, dtype=torch.float32, device=y.device)
        sums = torch.empty(N + t, dtype=torch.float32, device=y.device)
        _lib.check(lib.stl_token_fold_backward(g.data_ptr(), y.data_ptr(), B, Tp, N, t,
                                               fold32.data_ptr(), T, gy.data_ptr(),
                                               sums.data_ptr(), ws.data_ptr(), ws_n,
                                               _stream(y.device)))
        return gy, sums[N:], (sums[:N] if ctx.has_bias else None), None


class StlTokenLinear(nn.Module):
    """y = x W + b over token rows (B, T, in) with an STL layer (t, r).

    Weights are fake-encoded at init from a dense N(0, 1/in) matrix (toy_network.py:241-252:
    W_enc = encode_tiles(W0, e_w)); e_x, d, W_enc train, e_w stays fixed. T % t != 0 uses the
    paper's null-row padding and learnable fold of the last t rows.
    """

    def __init__(self, in_features: int, out_features: int, t: int = 4, r: int = 24,
                 init: str = "gaussian", bias: bool = True, seed: int = 0, device=None):
        super().__init__()
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.t, self.r = t, r
        self.in_features, self.out_features = in_features, out_features
        self.in_pad = -(-in_features // (8 * t)) * (8 * t) if in_features % t else in_features
        if out_features % t:
            raise ValueError(f"out_features {out_features} must be divisible by t={t}")
        snf = make_triple(t, r, init, seed).to(dev)
        w0 = torch.randn((self.in_pad, out_features), generator=torch.Generator().manual_seed(seed))
        w0 = (w0 / math.sqrt(in_features)).to(dev)
        w_enc = encode_tiles(w0, snf.e_w, t)                       # (in/t, out/t, r) fp32
        self.w_planes = nn.Parameter(weights_to_planes(w_enc, dtype=torch.float32).clone())
        self.e_x = nn.Parameter(snf.e_x.clone())
        self.d = nn.Parameter(snf.d.clone())
        self.bias = nn.Parameter(torch.zeros(out_features, device=dev)) if bias else None
        self.fold = nn.Parameter(torch.tensor([1.0] + [0.0] * (t - 1), device=dev))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        B, T, _ = x.shape
        t = self.t
        Tp = -(-T // t) * t
        if (Tp != T and T % t == 1 and self.in_features % 8 == 0 and self.in_pad % 8 == 0
                and self.out_features % 8 == 0 and x.is_cuda and FUSED_TOKEN_PLUMBING):
            # one-pass plumbing kernels: pad+cast in, fold+bias out (stl_tokens.cu)
            xp = TokenPad.apply(x, Tp, self.in_pad)
            y = StlLinearFunction.apply(xp.reshape(B * Tp, self.in_pad),
                                        self.w_planes.to(torch.bfloat16), self.e_x, self.d, t,
                                        self.r)
            return TokenFold.apply(y.reshape(B, Tp, self.out_features), self.fold, self.bias, T)
        x = x.to(torch.bfloat16)
        if self.in_pad != self.in_features:
            x = F.pad(x, (0, self.in_pad - self.in_features))
        t = self.t
        Tp = -(-T // t) * t
        folded = Tp != T
        if folded:
            if T % t != 1:
                raise ValueError(f"token count {T}: the fold supports T % t in (0, 1)")
            x = F.pad(x, (0, 0, 0, Tp - T))                       # null rows per sample
        y = StlLinearFunction.apply(x.reshape(B * Tp, self.in_pad).contiguous(),
                                    self.w_planes.to(torch.bfloat16), self.e_x, self.d, t, self.r)
        y = y.reshape(B, Tp, self.out_features)
        if folded:                                                # fold the last t rows into one
            last = torch.einsum("btn,t->bn", y[:, Tp - t:].float(), self.fold).to(y.dtype)
            y = torch.cat([y[:, :Tp - t], last[:, None]], dim=1)
        if self.bias is not None:
            y = y + self.bias.to(y.dtype)
        return y


def _linear(in_f, out_f, stl: bool, t, r, init, seed, bias=True, device=None):
    if stl:
        return StlTokenLinear(in_f, out_f, t, r, init, bias, seed, device)
    return nn.Linear(in_f, out_f, bias=bias, device=device)


class Attention(nn.Module):
    def __init__(self, dim, heads, stl, t, r, init, seed, device):
        super().__init__()
        self.heads = heads
        self.scale = (dim // heads) ** -0.5
        self.qkv = _linear(dim, 3 * dim, stl, t, r, init, seed, bias=False, device=device)
        self.proj = _linear(dim, dim, stl, t, r, init, seed + 1, device=device)

    def forward(self, x):
        B, T, C = x.shape
        qkv = self.qkv(x).reshape(B, T, 3, self.heads, C // self.heads).permute(2, 0, 3, 1, 4)
        y = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2], scale=self.scale)
        return self.proj(y.transpose(1, 2).reshape(B, T, C))


class Block(nn.Module):
    def __init__(self, dim, heads, mlp_ratio, stl, t, r, init, seed, device):
        super().__init__()
        self.norm1 = nn.LayerNorm(dim, device=device)
        self.attn = Attention(dim, heads, stl, t, r, init, seed, device)
        self.norm2 = nn.LayerNorm(dim, device=device)
        hidden = int(dim * mlp_ratio)
        self.fc1 = _linear(dim, hidden, stl, t, r, init, seed + 2, device=device)
        self.fc2 = _linear(hidden, dim, stl, t, r, init, seed + 3, device=device)

    def forward(self, x):
        x = x + self.attn(self.norm1(x))
        return x + self.fc2(F.gelu(self.fc1(self.norm2(x))))


class TokenPerformer(nn.Module):
    """T2T module's performer attention (Yuan et al. 2021, token_performer): linear-complexity
    attention with m = emb / 2 fixed orthogonal random features."""

    def __init__(self, dim, emb, stl, t, r, init, seed, device):
        super().__init__()
        self.emb = emb
        self.kqv = _linear(dim, 3 * emb, stl, t, r, init, seed, device=device)
        self.proj = _linear(emb, emb, stl, t, r, init, seed + 1, device=device)
        self.norm1 = nn.LayerNorm(dim, device=device)
        self.norm2 = nn.LayerNorm(emb, device=device)
        self.mlp1 = _linear(emb, emb, stl, t, r, init, seed + 2, device=device)
        self.mlp2 = _linear(emb, emb, stl, t, r, init, seed + 3, device=device)
        self.m = emb // 2
        w = torch.randn(self.m, emb, generator=torch.Generator().manual_seed(seed + 7))
        self.register_buffer("w", (torch.linalg.qr(w.T)[0].T * math.sqrt(self.m)).to(device))

    def prm_exp(self, x):
        xd = (x * x).sum(-1, keepdim=True) / 2
        return torch.exp(torch.einsum("bti,mi->btm", x.float(), self.w) - xd.float()) / math.sqrt(self.m)

    def forward(self, x):
        k, q, v = torch.split(self.kqv(self.norm1(x)), self.emb, dim=-1)
        kp, qp = self.prm_exp(k), self.prm_exp(q)
        D = torch.einsum("btm,bm->bt", qp, kp.sum(dim=1)).unsqueeze(-1)
        kptv = torch.einsum("bti,btm->bim", v.float(), kp)
        y = torch.einsum("btm,bim->bti", qp, kptv) / (D + 1e-8)
        y = v + self.proj(y.to(v.dtype))
        return y + self.mlp2(F.gelu(self.mlp1(self.norm2(y))))


def sinusoid_table(n, d):
    pos = np.arange(n)[:, None] / np.power(10000, 2 * (np.arange(d)[None] // 2) / d)
    pos[:, 0::2], pos[:, 1::2] = np.sin(pos[:, 0::2]), np.cos(pos[:, 1::2])
    return torch.tensor(pos, dtype=torch.float32)


def square_order(h: int, w: int, s: int = 2) -> torch.Tensor:
    """Permutation of the h x w raster patch order grouping every s x s square contiguously
    (PAPER.md:583)."""
    idx = torch.arange(h * w).reshape(h // s, s, w // s, s).permute(0, 2, 1, 3)
    return idx.reshape(-1)


class T2TViT7(nn.Module):
    """T2T-ViT-7: T2T module (performer, 7/4 -> 3/2 -> 3/2 soft splits, 64 channels), 196
    patch tokens + 1 class token, 7 blocks of dim 256 / 4 heads / MLP ratio 2, 1000 classes."""

    def __init__(self, num_classes=1000, stl=True, stl_t2t=False, t=4, r=24, init="gaussian",
                 img=224, device="cuda"):
        super().__init__()
        dev = torch.device(device)
        dim, t2t_dim = 256, 64
        self.t2t_1 = TokenPerformer(3 * 7 * 7, t2t_dim, stl_t2t, t, r, init, 100, dev)
        self.t2t_2 = TokenPerformer(t2t_dim * 9, t2t_dim, stl_t2t, t, r, init, 200, dev)
        self.project = _linear(t2t_dim * 9, dim, stl_t2t, t, r, init, 300, device=dev)
        self.grid = img // 16
        n = self.grid * self.grid
        self.register_buffer("order", square_order(self.grid, self.grid).to(dev))
        self.cls_token = nn.Parameter(torch.zeros(1, 1, dim, device=dev))
        self.register_buffer("pos", sinusoid_table(n + 1, dim)[None].to(dev))
        self.blocks = nn.ModuleList(
            [Block(dim, 4, 2.0, stl, t, r, init, 1000 + 10 * i, dev) for i in range(7)])
        self.norm = nn.LayerNorm(dim, device=dev)
        self.head = nn.Linear(dim, num_classes, device=dev)

    def forward(self, img):
        B = img.shape[0]
        with torch.autocast("cuda", dtype=torch.bfloat16):
            x = F.unfold(img, 7, stride=4, padding=2).transpose(1, 2)        # (B, 3136, 147)
            x = self.t2t_1(x)
            s = int(math.isqrt(x.shape[1]))
            x = F.unfold(x.transpose(1, 2).reshape(B, -1, s, s), 3, stride=2, padding=1).transpose(1, 2)
            x = self.t2t_2(x)
            s = int(math.isqrt(x.shape[1]))
            x = F.unfold(x.transpose(1, 2).reshape(B, -1, s, s), 3, stride=2, padding=1).transpose(1, 2)
            x = self.project(x)                                              # (B, 196, 256)
            x = x[:, self.order]                                             # 2x2 squares
            x = torch.cat([x, self.cls_token.expand(B, -1, -1).to(x.dtype)], dim=1) + self.pos
            for blk in self.blocks:
                x = blk(x)
            return self.head(self.norm(x)[:, -1])                            # class token


def allreduce_grads(params) -> None:
    """Average the gradients over the default process group in one flattened fp32 bucket
    (NCCL over NVLink for the GPU runs; any backend works)."""
    import torch.distributed as dist

    grads = [p.grad for p in params if p.grad is not None]
    if not grads:
        return
    flat = torch.cat([g.reshape(-1).float() for g in grads])
    dist.all_reduce(flat)
    flat /= dist.get_world_size()
    off = 0
    for g in grads:
        g.copy_(flat[off:off + g.numel()].view_as(g))
        off += g.numel()


def train_step(model, opt, img, labels, allreduce: bool = False):
    """One optimizer step (cross-entropy on the class token logits); with ``allreduce`` the
    gradients are averaged over the process group first (data parallel)."""
    opt.zero_grad(set_to_none=True)
    loss = F.cross_entropy(model(img).float(), labels)
    loss.backward()
    if allreduce:
        allreduce_grads(model.parameters())
    opt.step()
    return loss.detach()
