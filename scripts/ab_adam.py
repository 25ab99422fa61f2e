#!/usr/bin/env python3
"""A/B of ptk_chunk_adam between two builds of libptk (same box): one flat
chunk of N params, back-to-back launches between CUDA events, GB/s at 28 B/param.

    python scripts/ab_adam.py LIB.so [n_params] [reps]
"""
import ctypes
import sys

import torch

lib = ctypes.CDLL(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 268435456
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20


class Cfg(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("weight_decay", ctypes.c_double),
                ("adamw", ctypes.c_int32), ("step", ctypes.c_int32), ("grad_scale", ctypes.c_double)]


dev = torch.device("cuda", 0)
m = torch.zeros(n, dtype=torch.float32, device=dev)
v = torch.zeros_like(m)
p = torch.randn(n, device=dev) * 0.05
g = (torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16)
out = torch.empty(n, dtype=torch.bfloat16, device=dev)
lib.ptk_stats_workspace_bytes.restype = ctypes.c_int64
ws = torch.zeros(lib.ptk_stats_workspace_bytes(), dtype=torch.uint8, device=dev)
st = torch.zeros(2, dtype=torch.float64, device=dev)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
vp = lambda t: ctypes.c_void_p(t.data_ptr())
cfg = Cfg(1e-3, 0.9, 0.999, 1e-8, 0.0, 0, 1, 1.0)
for _ in range(3):
    assert lib.ptk_chunk_adam(ctypes.byref(cfg), vp(p), vp(m), vp(v), vp(g), vp(out), ctypes.c_int64(n),
                              vp(st), vp(ws), None, None, s) == 0
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lib.ptk_chunk_adam(ctypes.byref(cfg), vp(p), vp(m), vp(v), vp(g), vp(out), ctypes.c_int64(n),
                           vp(st), vp(ws), None, None, s)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / reps)
print(f"{sys.argv[1]} n={n} ms={best:.4f} GB/s={28 * n / best / 1e6:.1f}")
