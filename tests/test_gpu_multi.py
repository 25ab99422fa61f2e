"""Multi-GPU parity of the NCCL library path (one process per GPU, rank r on
cuda:r, NCCL over NVLink): ptk_chunk_reduce_scatter -> chunk Adam on the
owned shard -> ptk_chunk_allgather, and the N>1 bench flow with its training
leg. These run whenever the box has the GPUs and skip (with the reason) on
the one-GPU boxes of this build; the fused exchange across GPUs is in
test_gpu_ipc_fused.py.

Tolerance of NCCL's bf16 reduce-scatter: NCCL sums bf16 in
its ring order and rounds to bf16 after every hop, so per element
|rs - exact| <= (w - 1) * 2^-8 * sum_r |g_r| (one half-ulp of bf16 per hop,
bounded by the largest partial sum); the owned shard's Adam update from the
reduced gradient and the all-gather are bit-exact (the oracle is fed the
reduced bf16 shard the device produced).
"""
import ctypes
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle_lib as ol

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NUMELS = [1_000_003, 65_536]
STEPS = 3


def _need_gpus(n):
    have = torch.cuda.device_count()
    if have < n:
        pytest.skip(f"needs {n} GPUs (one NCCL rank per GPU), this box has {have}")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _nccl_rank(rank, world, port, out_dir, symmetric=False):
    import torch.distributed as dist
    sys.path.insert(0, REPO)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200 import chunks as ch
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    uid = (ctypes.c_uint8 * nat.PTK_UNIQUE_ID_BYTES)()
    if rank == 0:
        nat.lib.ptk_comm_unique_id(uid)
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
    dist.broadcast(t, 0)
    uid = (ctypes.c_uint8 * nat.PTK_UNIQUE_ID_BYTES)(*t.tolist())
    comm = ctypes.c_void_p()
    nat.lib.ptk_comm_init(ctypes.byref(comm), world, rank, uid)
    cs = ch.ChunkSet(NUMELS, world=world, rank=rank, device=dev, mode="nccl", comm=comm,
                     symmetric=symmetric)
    cs.init_synthetic()
    hyper = ch.AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True)
    s = torch.cuda.current_stream()
    out = {}
    for step in range(1, STEPS + 1):
        cs.fill_grads(step - 1, stream=s)
        cs.step(hyper, stream=s)
        nat.lib.ptk_comm_wait(comm, ch.stream_handle(s), 120_000)
        for c in cs.chunks:  # the reduce-scatter result, in place in this rank's shard
            red = c.grad[rank * c.shard:(rank + 1) * c.shard]
            out[f"red{c.chunk_id}_{step}"] = red.view(torch.int16).cpu().numpy().view(np.uint16)
    torch.cuda.synchronize()
    for c in cs.chunks:
        out[f"master{c.chunk_id}"] = c.master.cpu().numpy()
        out[f"param{c.chunk_id}"] = c.param.view(torch.int16).cpu().numpy().view(np.uint16)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
    dist.barrier()
    cs.close()   # collective: symmetric windows are deregistered on every rank
    nat.lib.ptk_comm_destroy(comm)
    dist.destroy_process_group()


def _spawn(world, tmp_path, symmetric=False):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_nccl_rank, args=(r, world, port, str(tmp_path), symmetric))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]


@pytest.mark.parametrize("symmetric", [False, True])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_rs_adam_ag_across_gpus(cuda_device, world, symmetric, tmp_path):
    """symmetric: chunk buffers in NCCL symmetric windows (ncclMemAlloc +
    ncclCommWindowRegister), the same stated bound."""
    from paper_2406_08334_b200 import chunks as ch
    _need_gpus(world)
    res = _spawn(world, tmp_path, symmetric)
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
                exact = sum(ol.bf16_to_f32(g[r * shard:(r + 1) * shard]).astype(np.float64)
                            for g in grads)
                mag = sum(np.abs(ol.bf16_to_f32(g[r * shard:(r + 1) * shard]).astype(np.float64))
                          for g in grads)
                red = res[r][f"red{ci}_{step}"]
                err = np.abs(ol.bf16_to_f32(red).astype(np.float64) - exact)
                assert np.all(err <= (world - 1) * 2.0 ** -8 * mag + 1e-30), float(err.max())
                ol.adam_step(ol.scalars(lr=1e-3, weight_decay=0.01, adamw=True, step=step,
                                        grad_scale=1.0 / world), mst, m, v, red, out)
            np.testing.assert_array_equal(res[r][f"master{ci}"].view(np.uint32), mst.view(np.uint32))
            params.append(out)
        gathered = ol.allgather(params)
        for r in range(world):
            np.testing.assert_array_equal(res[r][f"param{ci}"], gathered)


@pytest.mark.parametrize("world", [2, 8])
def test_bench_self_launch_across_gpus(cuda_device, world):
    """`bench.py --gpus N` on N real GPUs: self-launched ranks, both exchanges
    (fused over NVLink and NCCL) consistent across ranks, the NCCL training
    leg of the reference's test model (gpt2-1b b2) with a finite loss."""
    _need_gpus(world)
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["PTK_PEER_BARRIER_TIMEOUT_MS"] = "30000"
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", str(world),
                        "--workload", "cfg1", "--steps", "5", "--warmup", "3", "--train-steps", "3",
                        "--no-cpu-baseline", "--no-e2e"], capture_output=True, text=True,
                       timeout=1500, env=env, cwd=REPO)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    d = json.loads(lines[-1])
    assert d["n_gpus"] == world
    for leg in ("fused", "nccl"):
        assert d["exchanges"][leg]["consistent_across_ranks"] is True
    assert "error" not in d["train"] and np.isfinite(d["train"]["loss_last"])
