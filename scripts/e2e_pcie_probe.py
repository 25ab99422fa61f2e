import torch, ctypes, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2406_08334_b200 import _native as nat
dev = torch.device("cuda", 0)
TOT = 1557608000 // 2 * 2  # params
N = TOT
hg = torch.empty(N, dtype=torch.bfloat16, pin_memory=True)
hp = torch.empty(N, dtype=torch.bfloat16, pin_memory=True)
dg = torch.empty(N, dtype=torch.bfloat16, device=dev)
dp = torch.empty(N, dtype=torch.bfloat16, device=dev)
h2d, d2h, comp = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.current_stream()
def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(comp); h2d.wait_stream(comp); d2h.wait_stream(comp)
        fn()
        comp.wait_stream(h2d); comp.wait_stream(d2h); e1.record(comp)
        torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
def whole():
    with torch.cuda.stream(h2d): dg.copy_(hg, non_blocking=True)
    with torch.cuda.stream(d2h): hp.copy_(dp, non_blocking=True)
def pieces(p):
    def f():
        for lo in range(0, N, p):
            n = min(p, N - lo)
            with torch.cuda.stream(h2d): dg[lo:lo+n].copy_(hg[lo:lo+n], non_blocking=True)
            with torch.cuda.stream(d2h): hp[lo:lo+n].copy_(dp[lo:lo+n], non_blocking=True)
    return f
def chained(p, compute_ms=0.0):
    def f():
        for lo in range(0, N, p):
            n = min(p, N - lo)
            with torch.cuda.stream(h2d): dg[lo:lo+n].copy_(hg[lo:lo+n], non_blocking=True)
            e = torch.cuda.Event(); e.record(h2d); comp.wait_event(e)
            if compute_ms: nat.lib.ptk_busy_wait(int(compute_ms * 1e6 * n / N), ctypes.c_void_p(comp.cuda_stream))
            e2 = torch.cuda.Event(); e2.record(comp); d2h.wait_event(e2)
            with torch.cuda.stream(d2h): hp[lo:lo+n].copy_(dp[lo:lo+n], non_blocking=True)
    return f
print("whole", timed(whole))
for p in (1 << 22, 1 << 24, 1 << 25, 1 << 26, 1 << 27):
    print("pieces", p, timed(pieces(p)), "chained", timed(chained(p)), "chained+6.3ms compute", timed(chained(p, 6.3)))
