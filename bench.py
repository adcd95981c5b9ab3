#!/usr/bin/env python
"""bench.py — STL layer throughput on B200 (BASELINE.json metric, configs[1]).

A step = one STL linear layer forward + backward (all four gradients) at t=4, r=24, bf16,
M=8192 tokens, K=N=4096 (BASELINE configs[1]) on synthetic seeded data, through the C ABI
(stl_forward + stl_backward). Under torchrun every rank runs its own 8192-token batch
(data-parallel, weak scaling) and the gradients (g_w, g_ex, g_d) are all-reduced over NCCL
each step — the real exchange step of STL data-parallel training.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl stl|reference]

Prints ONE JSON line (rank 0). value = dense-equivalent TFLOP/s of the whole job
(3 * 2*M*K*N per rank per step / max-over-ranks device time). Inputs (~1 GB of live tensors per
step) are far larger than the 126 MB L2, so no explicit flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "STL layer dense-equiv TFLOP/s & speedup vs cuBLAS GEMM (t=4,r=24), at 1/2/4/8 B200"
UNIT = "TFLOP/s (dense-equivalent)"
T, R, M, K, N = 4, 24, 8192, 4096, 4096
WORKLOAD = "configs[1]: STL linear layer forward+backward t=4 r=24 bf16, M=8192 tokens, K=N=4096"


def dense_equiv_flops(m=M, k=K, n=N, passes=3):
    return passes * 2.0 * m * k * n


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_burst": d["bf16_tflops"],
                "bf16_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "bf16_burst": 1590.0, "bf16_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------------------- clocks
_SAMPLER_SRC = r"""
import sys, time
import pynvml as nv
nv.nvmlInit()
bus, path = sys.argv[1], sys.argv[2]
try:
    h = nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
except Exception:
    h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[3]))
fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
    getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
with open(path, "w") as f:
    print(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM), flush=True)
    while True:
        f.write(f"{time.time():.6f} {nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)} {fn(h)}\n")
        f.flush()
        time.sleep(0.002)
"""


class ClockSampler:
    """Polls NVML (SM clock, event reasons) every 2 ms in a CHILD process — a thread of this
    process would be starved by the launch loop holding the GIL — and keeps the samples taken
    between start() and stop()."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index: int):
        import subprocess
        import tempfile

        import torch
        self.max_mhz, self.proc = None, None
        self.path = tempfile.mktemp(prefix="stl_clocks_", suffix=".txt")
        try:
            props = torch.cuda.get_device_properties(device_index)
            bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
            self.proc = subprocess.Popen([sys.executable, "-c", _SAMPLER_SRC, bus, self.path,
                                          str(device_index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            line = self.proc.stdout.readline()  # max clock: the sampler is running
            self.max_mhz = int(line) if line.strip() else None
            if self.max_mhz is None:
                self.proc.kill()
                self.proc = None
        except Exception:  # noqa: BLE001 - clocks are reported as unavailable
            self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        self.t0 = time.time()

    def stop(self):
        self.t1 = time.time()
        samples, reasons = [], set()
        if self.proc is not None:
            time.sleep(0.005)
            self.proc.kill()
            self.proc.wait()
            try:
                with open(self.path) as f:
                    for line in f:
                        parts = line.split()
                        if len(parts) != 3 or not (self.t0 <= float(parts[0]) <= self.t1):
                            continue
                        samples.append(int(parts[1]))
                        for bit, name in self.REASONS.items():
                            if int(parts[2]) & bit:
                                reasons.add(name)
                os.unlink(self.path)
            except OSError:
                pass
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(samples)}


# ----------------------------------------------------------------------------- CPU baseline
def cpu_reference_step(rows: int, seed: int = 0):
    """The reference's CPU algorithm (oracle port, f64): stl forward (cached) + backward with
    the reference's own numpy call pattern (np.einsum without optimize), `rows` tokens."""
    from oracle import stl_oracle as O

    rng = O.make_rng(seed)
    e_x, e_w, d = O.random_gaussian_init(T, R, rng, scale=0.5)
    w_enc = O.encode_tiles(rng.standard_normal((K, N)) / np.sqrt(K), e_w, T)
    x = rng.standard_normal((rows, K))
    gy = rng.standard_normal((rows, N))

    def step():
        _y, cache = O.layer_forward_cached(x, w_enc, e_x, d, T)
        O.layer_backward_einsum(w_enc, e_x, d, cache, gy, T)

    return step


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, rank: int) -> None:
    """--impl reference: the reference's CPU implementation of the path (oracle port; the
    reference is pure Python and absent on the GPU box), rank 0 only."""
    if rank != 0:
        return
    rows = args.ref_rows
    step = cpu_reference_step(rows)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    sec = (time.perf_counter() - t0) / args.steps
    value = dense_equiv_flops(m=rows) / sec / 1e12
    sample = (f"{rows} of the 8192 tokens per step (K=N=4096, t=4, r=24, f64); forward "
              "stl_batched call pattern + backward np.einsum without optimize, as "
              "toy_network.py:95-106; numpy/OpenBLAS threads for the BLAS parts")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded PCG64)",
        "config": {"workload": WORKLOAD, "sample_rows": rows, "t": T, "r": R},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def rank_sweep(stl, lib, _lib, dev, stream, peaks, timed, n=8192, iters=5):
    """BASELINE configs[2]: forward at n^3, t in {2, 4}, r in {16, 24, 32, 49 (Strassen x
    Strassen)}; per point the forward time, its slice-GEMM rate against the burst bf16 peak and
    the transforms' HBM rate against the copy bandwidth (library profiler attribution)."""
    import torch

    x = torch.randn((n, n), device=dev).to(torch.bfloat16)
    out = []
    for t in (2, 4):
        for r in (16, 24, 32, 49):
            if r == 49 and t != 4:
                continue
            snf = (stl.strassen_rank49() if r == 49 else
                   stl.random_gaussian_init(t, r, stl.make_rng(0), scale=0.5)).to(dev)
            w = (torch.randn((r, n // t, n // t), device=dev) * 0.02).to(torch.bfloat16)
            u = torch.empty((r, n // t, n // t), dtype=torch.bfloat16, device=dev)
            sb = int(lib.stl_forward_scratch_bytes(n, n, n, t, r, _lib.STL_BF16))
            scratch = torch.empty((sb,), dtype=torch.uint8, device=dev)
            y = torch.empty((n, n), dtype=torch.bfloat16, device=dev)

            def fwd():
                _lib.check(lib.stl_forward(x.data_ptr(), n, n, n, w.data_ptr(), n,
                                           snf.e_x.data_ptr(), snf.d.data_ptr(), t, r,
                                           _lib.STL_BF16, y.data_ptr(), n, u.data_ptr(), None,
                                           scratch.data_ptr(), sb, stream))

            fwd()
            ms = timed(fwd, iters) / iters
            timed(fwd, iters, profile=True)
            recs = _lib.profile_records()
            g_ms = sum(m for nm, m, _ in recs if nm.startswith("slice_gemm")) / iters
            x_ms = sum(m for nm, m, _ in recs if nm in ("encode_x", "decode_y")) / iters
            p_bytes = 2 if r <= 32 else (3 if t == 4 else 4)  # bf16 / F24 / fp32 products
            cost = stl.LayerCost(n, n, n, t, r, 2, p_bytes)
            g_tf = cost.gemm_flops() / (g_ms * 1e-3) / 1e12
            xf_gbs = (cost.encode_bytes() + cost.decode_bytes()) / (x_ms * 1e-3) / 1e9
            out.append({"t": t, "r": r, "init": "strassen49" if r == 49 else "gaussian",
                        "fwd_ms": ms, "slice_gemm_tflops": g_tf,
                        "gemm_frac_of_burst": g_tf / peaks["bf16_burst"],
                        "transforms_GBs": xf_gbs, "transforms_hbm_frac": xf_gbs / peaks["hbm_gbs"],
                        "dense_over_stl_flops": 2 * n ** 3 / cost.forward_flops()})
            del w, u, scratch, y
            torch.cuda.empty_cache()
    return out


# ----------------------------------------------------------------------------- GPU arm
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("stl", "reference"), default="stl")
    ap.add_argument("--ref-rows", type=int, default=128)
    ap.add_argument("--cpu-rows", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip cuBLAS / 8192^3 / e2e legs")
    ap.add_argument("--no-t2t", action="store_true", help="skip the T2T-ViT-7 training leg")
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs[2] rank sweep")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks for exercising the multi-rank path on a one-GPU box: every rank on cuda:0, gloo
    if os.environ.get("STL_BENCH_SAME_DEVICE"):
        local = 0
    backend = os.environ.get("STL_BENCH_BACKEND", "nccl")

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2503_12211_b200 as stl
    from paper_2503_12211_b200 import _lib
    from paper_2503_12211_b200.layer import LayerCache, backward_raw
    from paper_2503_12211_b200.snf_operator import _forward

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    lib = _lib.load()
    peaks = load_peaks()

    # ---- problem: weights/encoders identical on every rank (DP replicas), data per rank
    rng = np.random.Generator(np.random.PCG64(0))
    snf = stl.random_gaussian_init(T, R, rng, scale=0.5).to(dev)
    w0 = torch.randn((K, N), generator=torch.Generator().manual_seed(1)) / K ** 0.5
    w_enc = stl.encode_tiles(w0.to(dev), snf.e_w, T)            # (bk, bj, r) fp32 view
    w_planes = stl.weights_to_planes(w_enc, dtype=torch.bfloat16)  # (r, bj, bk) bf16
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    x = torch.randn((M, K), device=dev, generator=g).to(torch.bfloat16)
    gy = torch.randn((M, N), device=dev, generator=g).to(torch.bfloat16)
    stl.set_check_finite(False)

    bi, bk, bj = M // T, K // T, N // T
    u = torch.empty((R, bi, bk), dtype=torch.bfloat16, device=dev)
    y_enc = torch.empty((int(lib.stl_cache_bytes(M, K, N, T, R, _lib.STL_BF16)),),
                        dtype=torch.uint8, device=dev)  # forward cache (slice products, AUTO format)
    fwd_scratch = torch.empty((int(lib.stl_forward_scratch_bytes(M, K, N, T, R, _lib.STL_BF16)),),
                              dtype=torch.uint8, device=dev)
    y = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    grads = torch.empty((R * bj * bk + 2 * R * T * T,), dtype=torch.float32, device=dev)
    g_w = grads[: R * bj * bk].view(R, bj, bk)
    g_ex = grads[R * bj * bk: R * bj * bk + R * T * T].view(R, T * T)
    g_d = grads[R * bj * bk + R * T * T:].view(R, T * T)
    g_x = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
    g_enc = torch.empty((R, bi, bj), dtype=torch.bfloat16, device=dev)
    g_u = torch.empty((R, bi, bk), dtype=torch.float32, device=dev)
    red = torch.empty((int(lib.stl_reduce_workspace_floats(R, T)),), dtype=torch.float32,
                      device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream

    cache_fmt = int(lib.stl_cache_format(M, K, N, T, R, _lib.STL_BF16, _lib.STL_PROD_AUTO))
    side = torch.cuda.Stream(dev)          # DP: g_w all-reduce beside the g_x / g_ex decode
    gw_ready = torch.cuda.Event()
    gw_ready.record()
    gw_done = torch.cuda.Event()

    def stl_step(allreduce: bool):
        _lib.check(lib.stl_forward(x.data_ptr(), M, K, K, w_planes.data_ptr(), N,
                                   snf.e_x.data_ptr(), snf.d.data_ptr(), T, R, _lib.STL_BF16,
                                   y.data_ptr(), N, u.data_ptr(), y_enc.data_ptr(),
                                   fwd_scratch.data_ptr(), fwd_scratch.numel(), stream))
        _lib.check(lib.stl_backward_ex(
            gy.data_ptr(), N, x.data_ptr(), K, w_planes.data_ptr(), snf.e_x.data_ptr(),
            snf.d.data_ptr(), u.data_ptr(), y_enc.data_ptr(), cache_fmt, M, K, N, T, R,
            _lib.STL_BF16, g_ex.data_ptr(), g_d.data_ptr(), g_w.data_ptr(), g_x.data_ptr(), K,
            g_enc.data_ptr(), g_u.data_ptr(), red.data_ptr(), _lib.STL_PROD_AUTO,
            gw_ready.cuda_event if allreduce else None, stream))
        if allreduce:
            # g_w (the bulk of the exchange) is final before the decode kernel: its NCCL
            # all-reduce runs on a side stream while decode_gu+g_ex computes; the small
            # encoder / decoder gradients follow on the main stream
            side.wait_event(gw_ready)
            with torch.cuda.stream(side):
                dist.all_reduce(g_w)
                gw_done.record(side)
            dist.all_reduce(grads[R * bj * bk:])
            torch.cuda.current_stream(dev).wait_event(gw_done)

    def timed(fn, steps, profile=False):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        if profile:
            lib.stl_profile_reset()
            lib.stl_profile_enable(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize(dev)
        if profile:
            lib.stl_profile_enable(0)
        ms = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
            dist.barrier()
        return ms

    # ---- warm-up, then the timed region (clocks sampled during it)
    for _ in range(args.warmup):
        stl_step(world > 1)
    torch.cuda.synchronize(dev)
    sampler = ClockSampler(local)
    sampler.start()
    total_ms = timed(lambda: stl_step(world > 1), args.steps)
    clocks = sampler.stop()
    ms_step = total_ms / args.steps
    value = world * dense_equiv_flops() / (ms_step * 1e-3) / 1e12

    # ---- per-kernel attribution: the same K steps again with the library's event profiler (CUDA
    # events around every launch on its stream). Kept out of the timed region above because
    # events between launches defeat programmatic dependent launch (+~7% step time).
    attr_ms = timed(lambda: stl_step(world > 1), args.steps, profile=True) / args.steps
    recs = _lib.profile_records()
    kern = {}
    launches = 0
    for name, ms, n in recs:
        k = kern.setdefault(name, {"ms": 0.0, "calls": 0})
        k["ms"] += ms
        k["calls"] += 1
        launches += n
    # bytes per stored slice product: the cache format (bf16 = 2, F24 = 3) on the bf16 path
    p_bytes = int(lib.stl_cache_bytes(M, K, N, T, R, _lib.STL_BF16)) // (R * bi * bj)
    cost = stl.LayerCost(M, K, N, T, R, 2, p_bytes)
    gem = kern.get("slice_gemm_tcgen05", {"ms": float("nan"), "calls": 1})
    # the step's three slice-GEMMs (y_enc forward; g_w and g_u backward, one grouped launch when
    # eligible) -> FLOP-weighted rate over all of the step's GEMM launches
    gemm_ms_step = gem["ms"] / args.steps
    gemm_flops_step = 3 * cost.gemm_flops()
    gemm_tflops = gemm_flops_step / (gemm_ms_step * 1e-3) / 1e12
    traffic = None
    tp = ROOT / "profiles" / "gemm_traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get("bytes_per_launch")
    # Denominator: the measured BURST bf16 peak when the timed region saw no power cap (short
    # regions run at full clock), the sustained peak when sw_power_cap was active.
    capped = "sw_power_cap" in (clocks.get("reasons") or [])
    peak = peaks["bf16_sustained"] if capped else peaks["bf16_burst"]
    roofline = {"kernel": "slice_gemm_tc2_kernel (CTA-pair tcgen05 slice GEMM; the step's 3 "
                          "slice-GEMMs over its launches, FLOP-weighted)", "bound": "tensor",
                "achieved": gemm_tflops, "peak": peak, "unit": "TFLOP/s",
                "frac": gemm_tflops / peak, "traffic": traffic,
                "traffic_of": "one forward slice-GEMM launch (ncu dram bytes)",
                "flops_per_step": gemm_flops_step, "ms_per_step": gemm_ms_step,
                "launches_per_step": gem["calls"] / args.steps,
                "frac_of_sustained": gemm_tflops / peaks["bf16_sustained"],
                "peak_source": peaks["source"] + (", sustained bf16 (sw_power_cap seen)" if capped
                                                  else ", burst bf16 (no power cap in the timed "
                                                       "region's clock samples)")}
    breakdown = {}
    step_kernel_ms = sum(v["ms"] for v in kern.values()) / args.steps
    hbm_bytes = {"encode_x": cost.encode_bytes(), "decode_y": cost.decode_bytes(),
                 "encode_gy+g_d": cost.encode_gy_gd_bytes(),
                 "decode_gu+g_ex": cost.decode_gu_gex_bytes()}
    for name, v in kern.items():
        per = v["ms"] / args.steps
        entry = {"ms_per_step": per, "share": per / step_kernel_ms if step_kernel_ms else None,
                 "calls_per_step": v["calls"] / args.steps}
        if name in hbm_bytes:
            gbs = hbm_bytes[name] / (v["ms"] / v["calls"] * 1e-3) / 1e9
            entry.update({"achieved_GBs": gbs, "hbm_frac": gbs / peaks["hbm_gbs"]})
        breakdown[name] = entry

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded randn; random-init N(0,0.25) encoders)",
        "config": {"workload": WORKLOAD, "M_per_rank": M, "K": K, "N": N, "t": T, "r": R,
                   "parallelism": f"dp{world}" if world > 1 else "single",
                   "l2": "inputs+intermediates ~1 GB/step > 126 MB L2 (no explicit flush)"},
        "roofline": roofline, "kernels": breakdown,
        "kernel_timing": {"how": "CUDA events around each launch (library profiler), separate "
                                 "pass of the same steps after the timed region",
                          "ms_per_step_with_events": attr_ms},
        "gpu_launches": launches, "clocks": clocks,
    }

    # ---- cuBLAS dense comparison on this rank (same shapes: Y=XW, dX=dY W^T, dW=X^T dY)
    if not args.no_extras:
        wd = torch.randn((K, N), device=dev).to(torch.bfloat16)
        yd = torch.empty((M, N), device=dev, dtype=torch.bfloat16)
        gxd = torch.empty((M, K), device=dev, dtype=torch.bfloat16)
        gwd = torch.empty((K, N), device=dev, dtype=torch.bfloat16)

        def dense_step():
            torch.matmul(x, wd, out=yd)
            torch.matmul(gy, wd.t(), out=gxd)
            torch.matmul(x.t(), gy, out=gwd)

        for _ in range(args.warmup):
            dense_step()
        # STL and cuBLAS timed in alternating blocks (same thermal / power state for both),
        # median block of each
        blk = max(args.steps // 4, 10)
        d_blocks, s_blocks = [], []
        for _ in range(5):
            s_blocks.append(timed(lambda: stl_step(False), blk) / blk)
            d_blocks.append(timed(dense_step, blk) / blk)
        dense_ms = statistics.median(d_blocks)
        stl_ms = statistics.median(s_blocks)
        line["vs_cublas"] = {"cublas_ms_per_step": dense_ms, "stl_ms_per_step": stl_ms,
                             "speedup": dense_ms / stl_ms, "timing": "5 alternating blocks of "
                             f"{blk} steps each (STL, cuBLAS), medians",
                             "cublas_tflops": dense_equiv_flops() / (dense_ms * 1e-3) / 1e12}
        del wd, yd, gxd, gwd

        # ---- north-star forward: 8192^3 bf16, t=4, r=24, STL forward vs cuBLAS forward.
        # Under torchrun (configs[4]) the 8192 token rows are sharded over the ranks with no
        # collective (rows of Y depend only on the same rows of X); time = max over ranks.
        n3 = 8192
        m_loc = n3 // world
        wf = stl.weights_to_planes(
            stl.encode_tiles(torch.randn((n3, n3), device=dev) / n3 ** 0.5, snf.e_w, T),
            dtype=torch.bfloat16)
        xf = torch.randn((m_loc, n3), device=dev).to(torch.bfloat16)
        uf = torch.empty((R, m_loc // T, n3 // T), dtype=torch.bfloat16, device=dev)
        sf = torch.empty((int(lib.stl_forward_scratch_bytes(m_loc, n3, n3, T, R, _lib.STL_BF16)),),
                         dtype=torch.uint8, device=dev)
        yf = torch.empty((m_loc, n3), dtype=torch.bfloat16, device=dev)
        wdf = torch.randn((n3, n3), device=dev).to(torch.bfloat16)
        ydf = torch.empty((m_loc, n3), device=dev, dtype=torch.bfloat16)

        def fwd8192():
            _lib.check(lib.stl_forward(xf.data_ptr(), m_loc, n3, n3, wf.data_ptr(), n3,
                                       snf.e_x.data_ptr(), snf.d.data_ptr(), T, R, _lib.STL_BF16,
                                       yf.data_ptr(), n3, uf.data_ptr(), None, sf.data_ptr(),
                                       sf.numel(), stream))

        steps_f = max(args.steps // 2, 10)
        for _ in range(args.warmup):
            fwd8192()
            torch.matmul(xf, wdf, out=ydf)
        # Burst (the north-star comparison, like MEASURED_PEAKS' burst GEMM): short alternating
        # blocks of 10 launches, each after 60 ms of idle so both run at their unthrottled clocks;
        # medians. Sustained: long alternating blocks back to back (both power-capped).
        def cub8192():
            torch.matmul(xf, wdf, out=ydf)

        sb_blocks, cb_blocks = [], []
        for _ in range(7):
            time.sleep(0.06)
            sb_blocks.append(timed(fwd8192, 10) / 10)
            time.sleep(0.06)
            cb_blocks.append(timed(cub8192, 10) / 10)
        sf_blocks, cf_blocks = [], []
        for _ in range(5):
            sf_blocks.append(timed(fwd8192, steps_f) / steps_f)
            cf_blocks.append(timed(cub8192, steps_f) / steps_f)
        stl_f = statistics.median(sb_blocks)
        timed(fwd8192, steps_f, profile=True)  # attribution pass (events between launches)
        recs_f = _lib.profile_records()
        gemm_f = [ms for name, ms, _ in recs_f
                  if name == "slice_gemm_tcgen05"]
        cub_f = statistics.median(cb_blocks)
        cost_f = stl.LayerCost(m_loc, n3, n3, T, R, 2, 2)
        gf_ms = sum(gemm_f) / max(len(gemm_f), 1)
        xf_ms = {n: sum(ms for nm, ms, _ in recs_f if nm == n) / steps_f
                 for n in ("encode_x", "decode_y")}
        gemm_tf = cost_f.gemm_flops() / (gf_ms * 1e-3) / 1e12
        line["north_star_fwd_8192"] = {
            "stl_ms": stl_f, "cublas_ms": cub_f, "speedup": cub_f / stl_f, "target": 1.8,
            "timing": "burst: 7 alternating blocks of 10 launches (STL forward, cuBLAS), each "
                      "after 60 ms idle, medians",
            "blocks_ms": {"stl": sb_blocks, "cublas": cb_blocks},
            "sustained": {"stl_ms": statistics.median(sf_blocks),
                          "cublas_ms": statistics.median(cf_blocks),
                          "speedup": statistics.median(cf_blocks) / statistics.median(sf_blocks),
                          "timing": f"5 alternating blocks of {steps_f} launches back to back "
                                    "(power-capped), medians"},
            "dense_equiv_tflops": 2 * n3 ** 3 / (stl_f * 1e-3) / 1e12,
            "m_sharded_over": world, "rows_per_rank": m_loc,
            "gemm_ms": gf_ms, "gemm_tflops": gemm_tf,
            "gemm_frac_of_burst": gemm_tf / peaks["bf16_burst"],
            "roofline": {
                "gemm": {"bound": "tensor", "achieved": gemm_tf, "peak": peaks["bf16_burst"],
                         "unit": "TFLOP/s", "frac": gemm_tf / peaks["bf16_burst"],
                         "flops_per_launch": cost_f.gemm_flops()},
                "encode_x": {"bound": "hbm", "bytes": cost_f.encode_bytes(),
                             "achieved": cost_f.encode_bytes() / (xf_ms["encode_x"] * 1e-3) / 1e9,
                             "peak": peaks["hbm_gbs"], "unit": "GB/s",
                             "frac": cost_f.encode_bytes() / (xf_ms["encode_x"] * 1e-3) / 1e9
                             / peaks["hbm_gbs"], "ms": xf_ms["encode_x"]},
                "decode_y": {"bound": "hbm", "bytes": cost_f.decode_bytes(),
                             "achieved": cost_f.decode_bytes() / (xf_ms["decode_y"] * 1e-3) / 1e9,
                             "peak": peaks["hbm_gbs"], "unit": "GB/s",
                             "frac": cost_f.decode_bytes() / (xf_ms["decode_y"] * 1e-3) / 1e9
                             / peaks["hbm_gbs"], "ms": xf_ms["decode_y"]},
                "how": "CUDA events around each launch (library profiler), attribution pass "
                       "after the timed region; peaks from MEASURED_PEAKS.json (burst bf16, "
                       "copy bandwidth)"},
        }
        del wf, xf, uf, sf, yf, wdf, ydf
        torch.cuda.empty_cache()

        # ---- configs[2]: rank / tile sweep of the forward at 8192^3 (rank 0; t = 2 slice
        # GEMMs are FLOP-losing by construction: the points report the fraction of roofline).
        if world == 1 and not args.no_sweep:
            line["rank_sweep"] = rank_sweep(stl, lib, _lib, dev, stream, peaks, timed)

        # ---- f1: a 3-layer bf16 chain at 8192^3 kept in encoded space (Algorithm 2) vs the
        # same layers as separate forwards (scripts/bench_chain.py; rank 0)
        if world == 1 and not args.no_sweep:
            sys.path.insert(0, str(Path(__file__).resolve().parent / "scripts"))
            from bench_chain import chain_bench
            line["fused_chain_8192"] = chain_bench()
            torch.cuda.empty_cache()

        # ---- e2e: public API (StlLinear autograd) with pinned host inputs, copies timed: a
        # training step's input is the batch X (the output gradient comes from the loss, here
        # L = ||Y||^2 / 2, so dY = Y, computed on the device), its result the loss and the
        # encoder / decoder gradients, read back every step. Double-buffered: step i's compute
        # overlaps the H2D copy of step i+1's batch on a copy stream (a data-loader prefetch).
        # Exactly one input copy per timed step is issued and consumed inside the timed region
        # (the pipeline is primed in the first timed step and the last step does not prefetch).
        mod = stl.StlLinear(snf, w_planes.clone())
        x_h = x.cpu().pin_memory()
        bufs = [(torch.empty_like(x),) for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_free = [torch.cuda.Event() for _ in range(2)]
        copy_s = torch.cuda.Stream(dev)
        out_h = torch.empty((2, R, T * T), dtype=torch.float32).pin_memory()
        loss_h = torch.empty((1,), dtype=torch.float32).pin_memory()
        pipe = {"i": 0, "left": 0}

        def issue_copy(slot):
            with torch.cuda.stream(copy_s):
                copy_s.wait_event(ev_free[slot])        # the step that last read it is done
                bufs[slot][0].copy_(x_h, non_blocking=True)
                ev_in[slot].record(copy_s)

        def e2e_step():
            i, slot = pipe["i"], pipe["i"] % 2
            if i == 0:
                issue_copy(slot)
            if pipe["left"] > 1:
                issue_copy(1 - slot)                     # prefetch step i+1
            cs = torch.cuda.current_stream(dev)
            cs.wait_event(ev_in[slot])
            x_d = bufs[slot][0]
            xin = x_d.detach().requires_grad_(True)
            mod.zero_grad(set_to_none=True)
            out = mod(xin)
            y = out.detach()
            loss = 0.5 * torch.linalg.vector_norm(y, dtype=torch.float32).square()
            out.backward(y)                              # dL/dY = Y
            if world > 1:
                dist.all_reduce(mod.w_planes.grad)
            loss_h.copy_(loss.reshape(1), non_blocking=True)
            out_h[0].copy_(mod.e_x.grad, non_blocking=True)
            out_h[1].copy_(mod.d.grad, non_blocking=True)
            ev_free[slot].record(cs)
            pipe["i"] += 1
            pipe["left"] -= 1

        def e2e_run(n):
            pipe.update(i=0, left=n)
            return lambda: e2e_step()

        steps_e = max(args.steps // 4, 10)
        run = e2e_run(args.warmup)
        for _ in range(args.warmup):
            run()
        torch.cuda.synchronize(dev)
        e2e_ms = timed(e2e_run(steps_e), steps_e) / steps_e
        line["e2e"] = {"value": world * dense_equiv_flops() / (e2e_ms * 1e-3) / 1e12,
                       "unit": UNIT, "ms_per_step": e2e_ms,
                       "h2d_bytes_per_step": x_h.numel() * 2,
                       "d2h_bytes_per_step": out_h.numel() * 4 + loss_h.numel() * 4,
                       "h2d_GBs": x_h.numel() * 2 / (e2e_ms * 1e-3) / 1e9,
                       "path": "StlLinear (autograd) training step: pinned host batch X copied "
                               "in (double-buffered on a copy stream), loss ||Y||^2/2 on the "
                               "device (dY = Y), forward+backward, loss and encoder/decoder "
                               "grads copied out each step"}

    # ---- configs[3] / configs[4]: T2T-ViT-7 training step with STL projections (trunk qkv,
    # proj, fc1, fc2 as STL r=24), synthetic 224x224, batch 256 per GPU, AdamW, gradient
    # all-reduce under torchrun; the dense nn.Linear model is timed the same way.
    if not args.no_extras and not args.no_t2t:
        from paper_2503_12211_b200 import t2t_vit

        res = {}
        for name, use_stl in (("stl_r24", True), ("dense", False)):
            torch.manual_seed(0)
            model = t2t_vit.T2TViT7(stl=use_stl, r=R, device=dev)
            opt = torch.optim.AdamW(model.parameters(), lr=1e-3, weight_decay=0.05)
            gen = torch.Generator(device=dev).manual_seed(rank)
            img = torch.randn(256, 3, 224, 224, device=dev, generator=gen)
            lab = torch.randint(0, 1000, (256,), device=dev, generator=gen)
            for _ in range(3):
                t2t_vit.train_step(model, opt, img, lab, allreduce=world > 1)
            ms = timed(lambda: t2t_vit.train_step(model, opt, img, lab, allreduce=world > 1), 5) / 5
            res[name] = {"ms_per_step": ms, "images_per_s": world * 256 / (ms * 1e-3),
                         "params": sum(p.numel() for p in model.parameters())}
            del model, opt, img, lab
            torch.cuda.empty_cache()
        line["t2t_vit7_train"] = {"batch_per_gpu": 256, **res,
                                  "note": "synthetic 224x224; STL layers memory-bound at these "
                                          "widths (K, N <= 768), see DESIGN"}

    # ---- CPU baseline (rank 0, N=1 only): the reference algorithm on a bounded sample
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows = args.cpu_rows
        step = cpu_reference_step(rows)
        runs = []
        for _ in range(3):  # best of 3
            t0 = time.perf_counter()
            step()
            runs.append(time.perf_counter() - t0)
        sec = min(runs)
        line["cpu_baseline"] = {
            "value": dense_equiv_flops(m=rows) / sec / 1e12, "unit": UNIT, "cores": cpu_cores(),
            "kind": "port",
            "sample": f"{rows} tokens x K=N=4096 fwd+bwd, f64, oracle port of stl_batched + "
                      f"_layer_backward (np.einsum as the reference), best of 3 runs "
                      f"({', '.join(f'{r:.1f}' for r in runs)} s)"}

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
