import torch, ctypes, sys, numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2406_08334_b200 import _native as nat
from paper_2406_08334_b200.chunks import vp
dev = torch.device("cuda", 0)
n = 512 * 1024 * 1024
master = torch.randn(n, device=dev) * 0.05
m = torch.zeros(n, device=dev); v = torch.zeros(n, device=dev)
g_dev = (torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16)
p_dev = torch.empty(n, dtype=torch.bfloat16, device=dev)
g_host = g_dev.cpu().pin_memory(); p_host = torch.empty(n, dtype=torch.bfloat16).pin_memory()
ws = torch.zeros(int(nat.raw.ptk_stats_workspace_bytes()), dtype=torch.uint8, device=dev)
stats = torch.zeros(2, dtype=torch.float64, device=dev)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
cfg = nat.adam_config(lr=1e-3, step=1)
def run(gp, pp, reps=3):
    best = 1e9
    for _ in range(reps):
        mm, mv, mv2 = master.clone(), m.clone(), v.clone()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = nat.raw.ptk_chunk_adam(ctypes.byref(cfg), vp(mm), vp(mv), vp(mv2), ctypes.c_void_p(gp), ctypes.c_void_p(pp), n, vp(stats), vp(ws), None, None, s)
        e1.record(); torch.cuda.synchronize()
        assert rc == 0, nat.last_error()
        best = min(best, e0.elapsed_time(e1))
    return best, mm
t_dev, ref = run(g_dev.data_ptr(), p_dev.data_ptr())
t_host, got = run(g_host.data_ptr(), p_host.data_ptr())
print("device ms", t_dev, "zero-copy ms", t_host, "GB/s PCIe each way", 2 * n / t_host / 1e6)
print("master equal", torch.equal(ref, got), "param equal", torch.equal(p_dev.cpu(), p_host))
t_r, _ = run(g_host.data_ptr(), p_dev.data_ptr())
t_w, _ = run(g_dev.data_ptr(), p_host.data_ptr())
print("zero-copy read-only ms", t_r, 2 * n / t_r / 1e6, "GB/s;  write-only ms", t_w, 2 * n / t_w / 1e6, "GB/s")
# write-only concurrently with a copy-engine H2D of another 1 GiB
big = torch.empty(n, dtype=torch.bfloat16).pin_memory(); bigd = torch.empty(n, dtype=torch.bfloat16, device=dev)
side = torch.cuda.Stream()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
e0.record(); side.wait_event(e0)
with torch.cuda.stream(side): bigd.copy_(big, non_blocking=True)
e2.record(side)
nat.raw.ptk_chunk_adam(ctypes.byref(cfg), vp(master), vp(m), vp(v), ctypes.c_void_p(g_dev.data_ptr()), ctypes.c_void_p(p_host.data_ptr()), n, vp(stats), vp(ws), None, None, s)
e1.record(); torch.cuda.synchronize()
print("write-only kernel with concurrent CE H2D: kernel", e0.elapsed_time(e1), "copy", e0.elapsed_time(e2))
