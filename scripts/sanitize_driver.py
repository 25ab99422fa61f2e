#!/usr/bin/env python3
"""Launch every libptk kernel once at small, ragged sizes (for
compute-sanitizer racecheck / synccheck / initcheck, scripts/sanitize.sh):
each chunk-Adam shape (TMA ring variants incl. the partial last tile, LDG),
the f32-grad variant, grad stats / prep, clip coefficient, the chunk-TABLE
launch (dynamic tile scheduler, several ragged chunks, back-to-back launches
re-arming the scheduler), the fused RS->Adam->AG kernel (TMA ring and
register-staged) over 2, 4 and 8 virtual ranks, the clipped fused step
(statistics pass, mailbox publish / collect), the peer barrier, fills."""
import ctypes
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet, vp
    dev = torch.device("cuda", 0)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    n = 3 * 148 * 2048 + 777          # several tiles per CTA plus a partial tile
    master = torch.empty(n, dtype=torch.float32, device=dev)
    m = torch.zeros_like(master)
    v = torch.zeros_like(master)
    g = torch.empty(n, dtype=torch.int16, device=dev)
    g32 = torch.empty(n, dtype=torch.float32, device=dev)
    p = torch.empty(n, dtype=torch.int16, device=dev)
    ws = torch.zeros(int(nat.raw.ptk_stats_workspace_bytes()), dtype=torch.uint8, device=dev)
    stats = torch.zeros(2, dtype=torch.float64, device=dev)
    nat.lib.ptk_fill_uniform_f32(vp(master), n, 1, 0, ctypes.c_float(0.05), s)
    nat.lib.ptk_fill_uniform_bf16(vp(g), n, 2, 0, ctypes.c_float(1e-3), s)
    cfg = nat.adam_config(lr=1e-3, weight_decay=0.01, adamw=True, step=1)
    nat.lib.ptk_stats_reset(vp(stats), s)
    nat.lib.ptk_chunk_adam(ctypes.byref(cfg), vp(master), vp(m), vp(v), vp(g), vp(p), n,
                           vp(stats), vp(ws), None, None, s)
    nat.lib.ptk_grad_prep(vp(g), n, ctypes.c_float(0.5), vp(g32), vp(stats), vp(ws), s)
    nat.lib.ptk_chunk_adam_f32grad(ctypes.byref(cfg), vp(master), vp(m), vp(v), vp(g32), vp(p),
                                   n, vp(stats), vp(ws), None, None, s)
    coef = torch.zeros(1, dtype=torch.float32, device=dev)
    skip = torch.zeros(1, dtype=torch.int32, device=dev)
    nat.lib.ptk_clip_coef(vp(stats), ctypes.c_double(1.0), vp(coef), vp(skip), s)
    nat.lib.ptk_chunk_adam(ctypes.byref(cfg), vp(master), vp(m), vp(v), vp(g), vp(p), n,
                           vp(stats), vp(ws), vp(coef), vp(skip), s)
    torch.cuda.synchronize()
    print("kernel shape in use:", nat.raw.ptk_adam_kernel_name().decode())

    # fused exchange over 2 virtual ranks + the peer barrier on one device
    sets = [ChunkSet([10_007, 4096], world=2, rank=r, device=dev, mode="fused") for r in range(2)]
    for cs in sets:
        cs.init_synthetic()
        cs.fill_grads(0)
        cs.attach_virtual_peers(sets)
    for cs in sets:
        cs.step(AdamHyper(lr=1e-3))
    # the TMA fused kernel at W = 4 (1536-element tiles) and W = 8 (1024):
    # several full tiles per rank + a partial tile
    for w, tile in ((4, 1536), (8, 1024)):
        sets_w = [ChunkSet([w * tile * 3 + 8 * w * 5], world=w, rank=r, device=dev, mode="fused")
                  for r in range(w)]
        for cs in sets_w:
            cs.init_synthetic()
            cs.fill_grads(0)
            cs.attach_virtual_peers(sets_w)
        for cs in sets_w:
            cs.step(AdamHyper(lr=1e-3))
    print("fused kernel in use:", nat.raw.ptk_fused_kernel_name().decode())

    # chunk-table launch: ragged chunks, tiles claimed dynamically, 3 launches
    # back to back (the last CTA re-arms the scheduler for the next launch)
    cs_t = ChunkSet([2048 * 150 + 8, 5000, 8, 2048 * 300 + 4096], device=dev)
    cs_t.init_synthetic()
    cs_t.fill_grads(0)
    for _ in range(3):
        cs_t.step(AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True))
    cs_t.step(AdamHyper(lr=1e-3), max_grad_norm=0.5, skip_nonfinite=True)

    # clipped fused step over virtual ranks: statistics pass, mailboxes, update
    from paper_2406_08334_b200.chunks import fused_group_step
    for w in (2, 4):
        sets_c = [ChunkSet([w * 2048 * 7 + 8 * w * 3, 4096], world=w, rank=r, device=dev,
                           mode="fused") for r in range(w)]
        for cs in sets_c:
            cs.init_synthetic()
            cs.fill_grads(0)
            cs.attach_virtual_peers(sets_c)
        fused_group_step(sets_c, AdamHyper(lr=1e-3), max_grad_norm=0.01, skip_nonfinite=True)
        fused_group_step(sets_c, AdamHyper(lr=1e-3))

    # the non-persistent chunks' peer exchange: fp32 peer reduce-scatter over
    # 3 virtual ranks' gradient chunks (ragged shard) + the copy-engine gather
    w, shard = 3, 2048 * 300 + 8
    gch = [torch.empty(w * shard, dtype=torch.int16, device=dev) for _ in range(w)]
    for r, t in enumerate(gch):
        nat.lib.ptk_fill_uniform_bf16(vp(t), w * shard, 40 + r, 0, ctypes.c_float(1e-3), s)
    red = torch.empty(shard, dtype=torch.float32, device=dev)
    gp = (ctypes.c_void_p * nat.PTK_MAX_PEERS)(*[t.data_ptr() for t in gch])
    for r in range(w):
        nat.lib.ptk_peer_reduce_scatter_f32(gp, w, r, shard, vp(red), s)
    nat.lib.ptk_peer_allgather(gp, w, 1, 2 * shard, s)

    # the register-staged fused kernel
    os.environ["PTK_FUSED_KERNEL"] = "ldg"
    sets_l = [ChunkSet([3 * 8 * 148 * 256 + 24], world=3, rank=r, device=dev, mode="fused")
              for r in range(3)]
    for cs in sets_l:
        cs.init_synthetic()
        cs.fill_grads(0)
        cs.attach_virtual_peers(sets_l)
    assert sets_l[0].fused_kernel == "ldg"
    for cs in sets_l:
        cs.step(AdamHyper(lr=1e-3))
    os.environ.pop("PTK_FUSED_KERNEL")
    sig = torch.zeros(nat.PTK_MAX_PEERS, dtype=torch.int32, device=dev)
    arr = (ctypes.c_void_p * nat.PTK_MAX_PEERS)(sig.data_ptr())
    nat.lib.ptk_peer_barrier(arr, 1, 0, 1, s)
    torch.cuda.synchronize()
    print("driver ok")


if __name__ == "__main__":
    main()
