"""World-size-2 and -3 coverage of the sharded (N>1) path on CPU with gloo.

Two processes each own half of a chunk (ptk_shard_elems mapping, padded to
8*w elements). Each produces its local gradients of the FULL chunk, the
gradients are reduce-scattered (gloo, fp32 sum), each rank updates its shard
with the product's host Adam (ptk_cpu_adam, K6 — the offloaded-chunk update of
the reference's CPU optimizer, proj/src/cost.cpp:213-218) using grad scale
1/w, and the bf16 shards are all-gathered. The gathered chunk and every shard
of master/m/v must be BIT-identical to a single-process oracle run over the
whole chunk with the summed gradients (same fp32 summation order: rank 0 then
rank 1).
"""
import ctypes
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = 10_001
STEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_08334_b200 import _native as nat
    import oracle_lib as ol
    shard = nat.shard_elems(N, world)
    n_pad = shard * world
    full_master = ol.fill_f32(n_pad, 0, 0.05)
    full_master[N:] = 0
    master = full_master[rank * shard:(rank + 1) * shard].copy()
    m = np.zeros(shard, np.float32)
    v = np.zeros(shard, np.float32)
    p_shard = np.zeros(shard, np.uint16)
    for step in range(1, STEPS + 1):
        g_local = ol.fill_bf16(n_pad, 1 + rank + 10 * step, 1e-3)
        g_local[N:] = 0
        g32 = torch.from_numpy(ol.bf16_to_f32(g_local).copy())
        out = torch.zeros(shard, dtype=torch.float32)
        if world == 2:
            dist.reduce_scatter(out, list(g32.split(shard)), op=dist.ReduceOp.SUM)
        else:
            # w > 2: gloo's ring sums in its own order; gather every rank's
            # owned slice and sum in rank order, the fused kernel's order
            parts = [torch.zeros(shard, dtype=torch.float32) for _ in range(world)]
            for r in range(world):
                slice_r = g32[r * shard:(r + 1) * shard].contiguous()
                dist.gather(slice_r, parts if r == rank else None, dst=r)
            out = parts[0].clone()
            for r in range(1, world):
                out += parts[r]
        # product host Adam takes bf16 grads: round the fp32 sum once (RS in bf16)
        g_shard = ol.f32_to_bf16(out.numpy())
        cfg = nat.adam_config(step=step, weight_decay=0.01, adamw=True, grad_scale=1.0 / world)
        nat.lib.ptk_cpu_adam(ctypes.byref(cfg), *[ctypes.c_void_p(x.ctypes.data)
                                                  for x in (master, m, v, g_shard, p_shard)],
                             shard, 1, None, None)
        # gloo has no 16-bit all-gather: move the bf16 bit patterns as int32
        gathered = [torch.zeros(shard, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(p_shard.astype(np.int32)))
    full = torch.cat(gathered).numpy().astype(np.uint16)
    np.save(os.path.join(outdir, f"rank{rank}.npy"), np.stack([master.view(np.uint32),
                                                                m.view(np.uint32),
                                                                v.view(np.uint32)]))
    np.save(os.path.join(outdir, f"params{rank}.npy"), full)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_step_equals_single_rank(tmp_path, world):
    import oracle_lib as ol
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    shard = ol.shard_elems(N, world)
    n_pad = shard * world
    master = ol.fill_f32(n_pad, 0, 0.05)
    master[N:] = 0
    m = np.zeros(n_pad, np.float32)
    v = np.zeros(n_pad, np.float32)
    out = np.zeros(n_pad, np.uint16)
    for step in range(1, STEPS + 1):
        grads = []
        for r in range(world):
            g = ol.fill_bf16(n_pad, 1 + r + 10 * step, 1e-3)
            g[N:] = 0
            grads.append(g)
        red = np.concatenate([ol.reduce_scatter(grads, r, shard) for r in range(world)])
        ol.adam_step(ol.scalars(step=step, weight_decay=0.01, adamw=True,
                                grad_scale=1.0 / world), master, m, v, red, out)
    for r in range(world):
        st = np.load(tmp_path / f"rank{r}.npy")
        sl = slice(r * shard, (r + 1) * shard)
        np.testing.assert_array_equal(st[0], master[sl].view(np.uint32))
        np.testing.assert_array_equal(st[1], m[sl].view(np.uint32))
        np.testing.assert_array_equal(st[2], v[sl].view(np.uint32))
        np.testing.assert_array_equal(np.load(tmp_path / f"params{r}.npy"), out)
    assert not out[N:].any()
