"""T2T-ViT-7 training step with STL projections (BASELINE configs[3]; configs[4] under torchrun).

    python scripts/bench_t2t.py [--batch 256] [--steps 10] [--warmup 3] [--r 24] [--dense]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/bench_t2t.py   # DP, NCCL

Synthetic 224x224 images and labels; a step = forward, cross-entropy, backward (STL layers
through the C ABI), gradient all-reduce over NCCL when WORLD_SIZE > 1, AdamW update. Prints one
JSON line: images/s (whole job, max-over-ranks device time) and ms per step.
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2503_12211_b200 import t2t_vit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256, help="images per GPU")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--r", type=int, default=24)
    ap.add_argument("--dense", action="store_true", help="dense nn.Linear baseline")
    ap.add_argument("--stl-t2t", action="store_true", help="STL in the T2T module too")
    ap.add_argument("--no-fused-tokens", action="store_true",
                    help="token pad/fold plumbing as framework ops (A/B)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.manual_seed(0)
    t2t_vit.FUSED_TOKEN_PLUMBING = not args.no_fused_tokens
    model = t2t_vit.T2TViT7(stl=not args.dense, stl_t2t=args.stl_t2t and not args.dense, r=args.r,
                            device=dev)
    opt = torch.optim.AdamW(model.parameters(), lr=1e-3, weight_decay=0.05)
    g = torch.Generator(device=dev).manual_seed(rank)
    img = torch.randn(args.batch, 3, 224, 224, device=dev, generator=g)
    labels = torch.randint(0, 1000, (args.batch,), device=dev, generator=g)
    for _ in range(args.warmup):
        t2t_vit.train_step(model, opt, img, labels, allreduce=world > 1)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        loss = t2t_vit.train_step(model, opt, img, labels, allreduce=world > 1)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    n_params = sum(p.numel() for p in model.parameters())
    if rank == 0:
        print(json.dumps({
            "workload": "T2T-ViT-7 training step, synthetic 224x224, AdamW"
                        + (" (dense baseline)" if args.dense else f", STL t=4 r={args.r} trunk"
                           + (" + T2T" if args.stl_t2t else "")),
            "n_gpus": world, "batch_per_gpu": args.batch, "ms_per_step": ms,
            "images_per_s": world * args.batch / (ms * 1e-3), "params": n_params,
            "loss": float(loss), "parallelism": f"dp{world}" if world > 1 else "single"}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
