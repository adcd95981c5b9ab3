"""CUDA-time breakdown of the T2T-ViT-7 training step (STL trunk vs dense) by kernel family."""
import json
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2503_12211_b200 import t2t_vit  # noqa: E402


def family(name: str) -> str:
    n = name.lower()
    if "k_stream" in n or "tiles_to_planes" in n or "planes_to_tiles" in n or "k_sum_partials" in n \
            or "transform" in n:
        return "stl_transform"
    if "slice_gemm" in n:
        return "stl_gemm"
    if "flash" in n or "fmha" in n or "attention" in n or "sdpa" in n:
        return "attention"
    if "gemm" in n or "cutlass" in n or "sm90" in n or "sm100" in n or "nvjet" in n:
        return "dense_gemm"
    if "adam" in n or "multi_tensor" in n:
        return "optimizer"
    if "conv" in n or "im2col" in n or "col2im" in n:
        return "conv/unfold"
    if "norm" in n:
        return "layernorm"
    return "elementwise/other"


def run(stl: bool, batch: int = 256):
    dev = torch.device("cuda")
    torch.manual_seed(0)
    model = t2t_vit.T2TViT7(stl=stl, r=24, device=dev)
    opt = torch.optim.AdamW(model.parameters(), lr=1e-3, weight_decay=0.05)
    img = torch.randn(batch, 3, 224, 224, device=dev)
    labels = torch.randint(0, 1000, (batch,), device=dev)
    for _ in range(3):
        t2t_vit.train_step(model, opt, img, labels)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            t2t_vit.train_step(model, opt, img, labels)
        torch.cuda.synchronize()
    fam = defaultdict(float)
    top = defaultdict(float)
    for e in prof.key_averages():
        if e.device_type.name != "CUDA":
            continue
        us = e.self_device_time_total / 3
        fam[family(e.key)] += us
        top[e.key[:90]] += us
    return {"stl": stl, "ms_total": sum(fam.values()) / 1e3,
            "families_ms": {k: round(v / 1e3, 3) for k, v in sorted(fam.items(), key=lambda x: -x[1])},
            "top": {k: round(v / 1e3, 3) for k, v in sorted(top.items(), key=lambda x: -x[1])[:25]}}


if __name__ == "__main__":
    for stl in (True, False):
        print(json.dumps(run(stl)))
