import torch, time
dev = torch.device("cuda", 0)
N = 1 << 29  # 512 Mi bf16 = 1 GiB
hg = torch.empty(N, dtype=torch.bfloat16, pin_memory=True)
hp = torch.empty(N, dtype=torch.bfloat16, pin_memory=True)
dg = torch.empty(N, dtype=torch.bfloat16, device=dev)
dp = torch.empty(N, dtype=torch.bfloat16, device=dev)
a = torch.empty(1 << 30, dtype=torch.float32, device=dev)
b = torch.empty_like(a)
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def run(hog_frac):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
    e0.record(s1); s2.wait_event(e0); s3.wait_event(e0)
    with torch.cuda.stream(s1): dg.copy_(hg, non_blocking=True)
    with torch.cuda.stream(s2): hp.copy_(dp, non_blocking=True)
    if hog_frac:
        with torch.cuda.stream(s3):
            for _ in range(hog_frac): b.copy_(a)
    e1.record(s1); e2.record(s2)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), e0.elapsed_time(e2)
for h in [0, 0, 10, 40, 0]:
    print("hog copies", h, "h2d/d2h ms", run(h))
# hog alone
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); [b.copy_(a) for _ in range(10)]; e1.record(); torch.cuda.synchronize(); print("10 hog copies alone ms", e0.elapsed_time(e1))
