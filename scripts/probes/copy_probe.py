"""Copy bandwidth of LDG/STG vs cp.async.bulk through shared memory (measurement aid)."""
import ctypes, json, os, sys
import torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libprobe.so"))
n = 1 << 30
a = torch.empty(n, dtype=torch.uint8, device="cuda"); b = torch.empty_like(a)
sms = torch.cuda.get_device_properties(0).multi_processor_count
for mode in (0, 1, 2):
    for _ in range(3): lib.probe_copy(mode, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_int64(n), sms, None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): lib.probe_copy(mode, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), ctypes.c_int64(n), sms, None)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"mode": ["ldg_stg", "bulk_1cta_per_sm", "bulk_2cta_per_sm"][mode], "GBs": 2 * n / ms / 1e6}))
ms_t = None
for _ in range(3): b.copy_(a)
torch.cuda.synchronize(); e0.record()
for _ in range(10): b.copy_(a)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"mode": "torch_copy", "GBs": 2 * n / (e0.elapsed_time(e1) / 10) / 1e6}))
