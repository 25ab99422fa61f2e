"""Multi-rank chunk training: ChunkedGPT2 over a world-w ChunkSet (ZeRO-3
chunk shards), each rank on its slice of one global batch, the
gradient exchange inside the training step.

* fused exchange, two or four PROCESSES on one GPU (runs on every box): each rank's
  parameters are views of its own chunk buffers; after the backward, the
  fused RS -> Adam -> AG kernel reads every rank's gradient chunk and writes
  every rank's parameter chunk through cudaIpc mappings (the NVLink code path
  with same-device memory). The result must equal, bit for bit, the same two
  ranks run as virtual ranks inside one process (the single-GPU validation
  of the exchange, tests/test_gpu_chunkset.py), with and without global-norm
  clipping; the replicas' gathered parameters must be identical; and the
  loss trajectory must follow the w=1 run on the whole global batch.
* NCCL exchange and the non-persistent chunk pool at w=2 (one rank per GPU,
  skipped with the reason on one-GPU boxes): replicas identical, pooled
  (host Adam, NCCL reduce-scatter in ChunkGather.backward, all-gather on
  fetch) bit-identical to all-persistent at the same w, losses following w=1.

The reference models these exchanges as gather_time / reduce_time
(proj/src/hardware.cpp:29-38) and the simulator's Gather / Reduce phases
(proj/src/sim.cpp:335-350,426-436).
"""
import json
import os
import socket
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SPEC = {"hidden_size": 256, "n_blocks": 2, "n_heads": 4, "vocab_size": 1000, "seq_len": 128}
GLOBAL_BATCH = 4
STEPS = 3


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _need_gpus(n):
    have = torch.cuda.device_count()
    if have < n:
        pytest.skip(f"needs {n} GPUs (one NCCL rank per GPU), this box has {have}")


def _build(d: Path, dev, world, rank, mode, comm=None, n_persist=None, n_buffer=0,
           pool_exchange=None):
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import ChunkSet
    from paper_2406_08334_b200.offload import ChunkPool
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape
    d.mkdir(parents=True, exist_ok=True)
    spec = d / "spec.json"
    spec.write_text(json.dumps(SPEC))
    tpath = planner.trace_file(["--spec", str(spec), "--batch", str(GLOBAL_BATCH)], str(d / "t.json"))
    trace = json.load(open(tpath))
    layout = planner.pack(tpath, grid="2Mi")
    numels = [c["used_bytes"] // 2 for c in layout["chunks"]]
    np_ = len(numels) if n_persist is None else n_persist
    cs = ChunkSet(numels[:np_], world=world, rank=rank, device=dev, mode=mode, comm=comm)
    # the fused exchange's pool exchanges over peer memory too (no NCCL)
    pool = (ChunkPool(numels, np_, n_buffer, world=world, rank=rank, comm=comm, device=dev,
                      piece=65_544,
                      exchange=pool_exchange or ("peer" if mode == "fused" else "nccl"))
            if np_ < len(numels) else None)
    shape = GPT2Shape.from_trace_meta(trace["meta"], trace["n_blocks"])
    model = ChunkedGPT2(shape, layout, cs, trace["ops"], pool=pool)
    model.init_weights(seed=0)
    return model, shape, numels


def _batches(shape, dev):
    """The global batch of every step (identical on every rank)."""
    g = torch.Generator(device=dev).manual_seed(0)
    for _ in range(STEPS):
        x = torch.randint(0, shape.vocab, (GLOBAL_BATCH, shape.seq), device=dev, generator=g)
        yield x, (x + 1) % shape.vocab


def _hyper():
    from paper_2406_08334_b200.chunks import AdamHyper
    return AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True)


def _state(model, numels):
    """Gathered bf16 parameters and this rank's fp32 master shard per chunk."""
    out = {}
    for c in model.chunks.chunks:
        out[f"param{c.chunk_id}"] = c.param[:c.numel].view(torch.int16).cpu().numpy()
        out[f"master{c.chunk_id}"] = c.master.cpu().numpy().view(np.uint32)
    pool = model.pool
    if pool is not None:
        pool.finish_step()
        for c in sorted(pool.numel):
            out[f"master{c}"] = pool.h_master[c].numpy().view(np.uint32).copy()
            out[f"hparam{c}"] = pool.h_param[c].view(torch.int16).numpy().copy()
    return out


def _rank_main(rank, world, port, out_dir, mode, spread, max_norm, n_persist, n_buffer,
               overlap=False):
    import ctypes

    import torch.distributed as dist
    os.environ["PTK_PEER_BARRIER_TIMEOUT_MS"] = "60000"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2406_08334_b200 import _native as nat
    from paper_2406_08334_b200.train import train_step
    dev = torch.device("cuda", rank if spread else 0)
    torch.cuda.set_device(dev)
    comm = None
    if mode == "nccl":
        uid = (ctypes.c_uint8 * nat.PTK_UNIQUE_ID_BYTES)()
        if rank == 0:
            nat.lib.ptk_comm_unique_id(uid)
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
        dist.broadcast(t, 0)
        uid = (ctypes.c_uint8 * nat.PTK_UNIQUE_ID_BYTES)(*t.tolist())
        comm = ctypes.c_void_p()
        nat.lib.ptk_comm_init(ctypes.byref(comm), world, rank, uid)
    model, shape, numels = _build(Path(out_dir) / f"r{rank}", dev, world, rank, mode, comm,
                                  n_persist, n_buffer)
    if mode == "fused":
        model.chunks.attach_ipc_peers()
        if model.pool is not None:
            model.pool.attach_ipc_peers()
    hyper = _hyper()
    b = GLOBAL_BATCH // world
    losses = []
    for x, y in _batches(shape, dev):
        xs, ys = x[rank * b:(rank + 1) * b], y[rank * b:(rank + 1) * b]
        if max_norm > 0:
            loss = model.loss(xs, ys)
            loss.backward()
            model.chunks.step(hyper, max_grad_norm=max_norm)
        else:
            loss = train_step(model, xs, ys, hyper, overlap=overlap)
        losses.append(float(loss.detach()))
    torch.cuda.synchronize()
    out = _state(model, numels)
    out["losses"] = np.array(losses, np.float64)
    out["coef"] = np.array([float(model.chunks.clip_coef[0])], np.float32)
    dist.barrier()   # nobody unmaps / destroys while a peer may still use it
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
    if mode == "fused":
        model.chunks.close_ipc_peers()
        if model.pool is not None:
            model.pool.close_ipc_peers()
    if comm is not None:
        nat.lib.ptk_comm_destroy(comm)
    dist.destroy_process_group()


def _spawn(world, tmp_path, mode, spread=False, max_norm=0.0, n_persist=None, n_buffer=0,
           overlap=False):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    out = tmp_path / f"{mode}_{n_persist}_{max_norm}_{overlap}"
    out.mkdir(parents=True, exist_ok=True)
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, str(out), mode, spread,
                                                  max_norm, n_persist, n_buffer, overlap))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=400)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return [dict(np.load(out / f"rank{r}.npz")) for r in range(world)]


def _virtual(tmp_path, dev, world, max_norm):
    """The same w ranks as virtual ranks of one process on one device."""
    from paper_2406_08334_b200.chunks import fused_group_step
    models = [_build(tmp_path / f"virtual{r}", dev, world, r, "fused")[0] for r in range(world)]
    shape = models[0].shape
    sets = [m.chunks for m in models]
    for cs in sets:
        cs.attach_virtual_peers(sets)
    b = GLOBAL_BATCH // world
    losses = [[] for _ in range(world)]
    for x, y in _batches(shape, dev):
        for r, m in enumerate(models):
            loss = m.loss(x[r * b:(r + 1) * b], y[r * b:(r + 1) * b])
            loss.backward()
            losses[r].append(float(loss.detach()))
        fused_group_step(sets, _hyper(), max_grad_norm=max_norm)
    torch.cuda.synchronize()
    res = []
    for r, m in enumerate(models):
        out = _state(m, None)
        out["losses"] = np.array(losses[r], np.float64)
        out["coef"] = np.array([float(m.chunks.clip_coef[0])], np.float32)
        res.append(out)
    return res


def _w1_losses(tmp_path, dev):
    from paper_2406_08334_b200.train import train_step
    model, shape, _ = _build(tmp_path / "w1", dev, 1, 0, "nccl")
    return [float(train_step(model, x, y, _hyper())) for x, y in _batches(shape, dev)]


def _replicas_identical(res):
    for k in res[0]:
        if k.startswith("param"):
            for r in range(1, len(res)):
                np.testing.assert_array_equal(res[r][k], res[0][k], err_msg=k)


def _follows_w1(res, w1):
    # mean of the ranks' local losses (each over GLOBAL_BATCH / w sequences)
    # against the w=1 loss over the whole batch: same data, same update up to
    # the gradient's rounding (per-rank bf16 gradients summed in fp32)
    mean = np.mean([r["losses"] for r in res], axis=0)
    np.testing.assert_allclose(mean, w1, rtol=2e-3)
    assert mean[-1] < mean[0]


@pytest.mark.parametrize("world,max_norm", [(2, 0.0), (2, 0.05), (4, 0.0)])
def test_fused_training_processes_equal_virtual_ranks(tmp_path, cuda_device, world, max_norm):
    res = _spawn(world, tmp_path, "fused", max_norm=max_norm)
    ref = _virtual(tmp_path, cuda_device, world, max_norm)
    for r in range(world):
        for k, v in ref[r].items():
            np.testing.assert_array_equal(res[r][k], v, err_msg=f"rank {r} {k}")
    _replicas_identical(res)
    if max_norm > 0:
        assert res[0]["coef"][0] < 1.0   # the clip engaged (same coefficient on every rank)
        assert all(r["coef"][0] == res[0]["coef"][0] for r in res)
    else:
        _follows_w1(res, _w1_losses(tmp_path, cuda_device))
        assert res[0]["losses"].size == STEPS


def test_fused_overlapped_training_equals_fused(tmp_path, cuda_device):
    """overlap=True with the fused exchange (two processes on this GPU): each
    chunk's reduce runs on a side stream as soon as its gradients are complete
    (peer reduce-scatter between barriers, overlapping the rest of the
    backward), the Adam on the fp32 reduced shards and the all-gather follow
    the backward -- bit-identical to the one-kernel fused step."""
    world = 2
    ref = _spawn(world, tmp_path, "fused")
    res = _spawn(world, tmp_path, "fused", overlap=True)
    for r in range(world):
        for k, v in ref[r].items():
            if k != "coef":
                np.testing.assert_array_equal(res[r][k], v, err_msg=f"rank {r} {k}")


def test_peer_pool_single_rank_equals_persistent(tmp_path, cuda_device):
    """exchange='peer' at w = 1: the offloaded chunk's gradient goes to the
    host as fp32 and the host Adam runs on it -- the same numbers as the
    device Adam on the bf16 gradient, so losses and masters equal the
    all-persistent run bit for bit."""
    from paper_2406_08334_b200.train import train_step
    runs = []
    for n_persist, n_buffer in ((None, 0), (1, 1)):
        model, shape, numels = _build(tmp_path / f"w1peer_{n_persist}", cuda_device, 1, 0,
                                      "nccl", n_persist=n_persist, n_buffer=n_buffer,
                                      pool_exchange="peer")
        if model.pool is not None:
            assert model.pool.h_grad[1].dtype == torch.float32
        losses = [float(train_step(model, x, y, _hyper()).detach())
                  for x, y in _batches(shape, cuda_device)]
        torch.cuda.synchronize()
        st = _state(model, numels)
        runs.append((losses, {k: v for k, v in st.items() if k.startswith("master")}))
    assert runs[0][0] == runs[1][0]
    for k, v in runs[0][1].items():
        np.testing.assert_array_equal(runs[1][1][k][:v.size], v, err_msg=k)


def test_peer_pool_two_processes_equals_persistent(tmp_path, cuda_device):
    """w = 2 in two processes on this GPU, NO library collective anywhere:
    chunk 0 persistent (fused RS->Adam->AG), chunks 1-2 non-persistent in a
    one-slot pool that gathers over peer memory (copy-engine pulls between
    peer barriers) and drains through the fp32 peer reduce-scatter into the
    host Adam. Losses and every master shard equal the all-persistent fused
    run bit for bit (same fp32 rank-order sums, same update rule)."""
    world = 2
    ref = _spawn(world, tmp_path, "fused")
    res = _spawn(world, tmp_path, "fused", n_persist=1, n_buffer=1)
    for r in range(world):
        np.testing.assert_array_equal(res[r]["losses"], ref[r]["losses"])
        for k, v in ref[r].items():
            if k.startswith("master"):
                np.testing.assert_array_equal(res[r][k][:v.size], v, err_msg=f"rank {r} {k}")


def test_fused_and_peer_pool_training_across_gpus(tmp_path, cuda_device):
    """The same checks with one rank per GPU (NVLink peers): fused training
    equals the virtual-rank run, and the peer pool and the overlapped fused
    step equal the all-persistent fused run, bit for bit."""
    world = 2
    _need_gpus(world)
    ref = _spawn(world, tmp_path, "fused", spread=True)
    virt = _virtual(tmp_path, cuda_device, world, 0.0)
    for r in range(world):
        for k, v in virt[r].items():
            np.testing.assert_array_equal(ref[r][k], v, err_msg=f"rank {r} {k}")
    res = _spawn(world, tmp_path / "pool", "fused", spread=True, n_persist=1, n_buffer=1)
    for r in range(world):
        np.testing.assert_array_equal(res[r]["losses"], ref[r]["losses"])
        for k, v in ref[r].items():
            if k.startswith("master"):
                np.testing.assert_array_equal(res[r][k][:v.size], v, err_msg=f"rank {r} {k}")
    ov = _spawn(world, tmp_path / "overlap", "fused", spread=True, overlap=True)
    for r in range(world):
        for k, v in ref[r].items():
            if k != "coef":
                np.testing.assert_array_equal(ov[r][k], v, err_msg=f"overlap rank {r} {k}")


def test_nccl_training_across_gpus(tmp_path, cuda_device):
    world = 2
    _need_gpus(world)
    res = _spawn(world, tmp_path, "nccl", spread=True)
    _replicas_identical(res)
    _follows_w1(res, _w1_losses(tmp_path, cuda_device))


def test_pooled_training_across_gpus_equals_persistent(tmp_path, cuda_device):
    """Non-persistent chunks at w=2 (ChunkPool: NCCL reduce-scatter of the
    drained gradient, host Adam on the rank's shard, H2D + all-gather on
    fetch) give the all-persistent NCCL run's losses and masters bit for bit
    (host Adam == device Adam; the same NCCL reduce-scatter)."""
    world = 2
    _need_gpus(world)
    ref = _spawn(world, tmp_path, "nccl", spread=True)
    res = _spawn(world, tmp_path, "nccl", spread=True, n_persist=1, n_buffer=1)
    for r in range(world):
        np.testing.assert_array_equal(res[r]["losses"], ref[r]["losses"])
        for k, v in ref[r].items():
            if k.startswith("master"):
                np.testing.assert_array_equal(res[r][k][:v.size], v, err_msg=f"rank {r} {k}")
