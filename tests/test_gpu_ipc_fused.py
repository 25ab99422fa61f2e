"""The multi-process fused exchange (ptk_fused_rs_adam_ag over cudaIpc peer
mappings + ptk_peer_barrier) with REAL separate processes.

The GPU tiers here have one GPU, so both ranks live on cuda:0: each process
maps the other's gradient / parameter chunks and signal slots through
cudaIpc handles exactly as on an NVLink node (same code path:
ChunkSet.attach_ipc_peers -> ptk_ipc_open_handle), exchanging the handles
over a gloo group. Only the wire differs (same-device memory instead of
NVLink). The results must equal the oracle bit for bit, like the
virtual-rank test in test_gpu_chunkset.py.
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle_lib as ol

pytestmark = pytest.mark.gpu

NUMELS = [10_007, 4096]
STEPS = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["PTK_PEER_BARRIER_TIMEOUT_MS"] = "20000"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2406_08334_b200 import chunks as ch
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cs = ch.ChunkSet(NUMELS, world=world, rank=rank, device=dev, mode="fused")
    cs.init_synthetic()
    cs.fill_grads(0)
    torch.cuda.synchronize()
    cs.attach_ipc_peers()
    hyper = ch.AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True)
    s = torch.cuda.current_stream()
    for step in range(1, STEPS + 1):
        cs.step(hyper, stream=s)
        if step < STEPS:
            cs.fill_grads(step, stream=s)   # after the closing barrier: peers are done reading
    torch.cuda.synchronize()
    dist.barrier()   # nobody unmaps while a peer may still store into it
    out = {}
    for c in cs.chunks:
        out[f"master{c.chunk_id}"] = c.master.cpu().numpy()
        out[f"m{c.chunk_id}"] = c.exp_avg.cpu().numpy()
        out[f"v{c.chunk_id}"] = c.exp_avg_sq.cpu().numpy()
        out[f"param{c.chunk_id}"] = c.param.view(torch.int16).cpu().numpy().view(np.uint16)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
    cs.close_ipc_peers()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_across_processes_bit_exact(cuda_device, world, tmp_path):
    import torch.multiprocessing as mp
    from paper_2406_08334_b200 import chunks as ch
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, str(tmp_path)))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for ci, n in enumerate(NUMELS):
        shard = ol.shard_elems(n, world)
        n_pad = shard * world
        master_full = ol.fill_f32(n_pad, ch.master_seed(ci), ch.MASTER_SCALE)
        master_full[n:] = 0
        params = []
        for r in range(world):
            mst = master_full[r * shard:(r + 1) * shard].copy()
            m = np.zeros(shard, np.float32)
            v = np.zeros(shard, np.float32)
            out = np.zeros(shard, np.uint16)
            for step in range(1, STEPS + 1):
                grads = []
                for q in range(world):
                    g = ol.fill_bf16(n_pad, ch.grad_seed(ci, q, step - 1), ch.GRAD_SCALE)
                    g[n:] = 0
                    grads.append(g)
                red = ol.reduce_scatter(grads, r, shard, fp32=True)
                ol.adam_step(ol.scalars(lr=1e-3, weight_decay=0.01, adamw=True, step=step,
                                        grad_scale=1.0 / world), mst, m, v, red, out)
            np.testing.assert_array_equal(res[r][f"master{ci}"].view(np.uint32), mst.view(np.uint32))
            np.testing.assert_array_equal(res[r][f"m{ci}"].view(np.uint32), m.view(np.uint32))
            np.testing.assert_array_equal(res[r][f"v{ci}"].view(np.uint32), v.view(np.uint32))
            params.append(out)
        gathered = ol.allgather(params)
        for r in range(world):
            np.testing.assert_array_equal(res[r][f"param{ci}"], gathered)
