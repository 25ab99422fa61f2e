"""The multi-process fused exchange (ptk_fused_rs_adam_ag over cudaIpc peer
mappings + ptk_peer_barrier) with REAL separate processes.

The GPU tiers here have one GPU, so the `shared` tests put every rank on
cuda:0: each process maps the other's gradient / parameter chunks and signal
slots through cudaIpc handles exactly as on an NVLink node (same code path:
ChunkSet.attach_ipc_peers -> ptk_ipc_open_handle), exchanging the handles
over a gloo group. Only the wire differs (same-device memory instead of
NVLink). The `spread` tests put rank r on cuda:r -- the real NVLink path,
both fused kernels (TMA ring and register-staged) -- and run whenever the
box has enough GPUs (skipped, with the reason, on one-GPU boxes). The
results must equal the oracle bit for bit, like the virtual-rank test in
test_gpu_chunkset.py.
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


def _rank_main(rank, world, port, out_dir, max_norm=0.0, spread=False, kernel=""):
    import torch.distributed as dist
    os.environ["PTK_PEER_BARRIER_TIMEOUT_MS"] = "20000"
    if kernel:
        os.environ["PTK_FUSED_KERNEL"] = kernel
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2406_08334_b200 import chunks as ch
    dev = torch.device("cuda", rank if spread else 0)
    torch.cuda.set_device(dev)
    cs = ch.ChunkSet(NUMELS, world=world, rank=rank, device=dev, mode="fused")
    cs.init_synthetic()
    cs.fill_grads(0)
    torch.cuda.synchronize()
    cs.attach_ipc_peers()
    hyper = ch.AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True)
    s = torch.cuda.current_stream()
    coefs = []
    for step in range(1, STEPS + 1):
        cs.step(hyper, stream=s, max_grad_norm=max_norm)
        coefs.append(float(cs.clip_coef[0]))  # host sync: this step's device coefficient
        if step < STEPS:
            cs.fill_grads(step, stream=s)   # after the closing barrier: peers are done reading
    torch.cuda.synchronize()
    dist.barrier()   # nobody unmaps while a peer may still store into it
    out = {"coef": np.array(coefs, np.float32), "kernel": np.array([cs.fused_kernel])}
    for c in cs.chunks:
        out[f"master{c.chunk_id}"] = c.master.cpu().numpy()
        out[f"m{c.chunk_id}"] = c.exp_avg.cpu().numpy()
        out[f"v{c.chunk_id}"] = c.exp_avg_sq.cpu().numpy()
        out[f"param{c.chunk_id}"] = c.param.view(torch.int16).cpu().numpy().view(np.uint16)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
    cs.close_ipc_peers()
    dist.destroy_process_group()


def _spawn(world, tmp_path, max_norm=0.0, spread=False, kernel=""):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank_main,
                         args=(r, world, port, str(tmp_path), max_norm, spread, kernel))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    for p in procs:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]


def _need_gpus(n):
    have = torch.cuda.device_count()
    if have < n:
        pytest.skip(f"needs {n} GPUs (NVLink peers), this box has {have}")


def _check_fused(res, world):
    from paper_2406_08334_b200 import chunks as ch
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


@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_across_processes_bit_exact(cuda_device, world, tmp_path):
    res = _spawn(world, tmp_path)
    assert all(str(r["kernel"][0]) == "tma" for r in res)  # the default: the TMA ring
    _check_fused(res, world)


@pytest.mark.parametrize("kernel", ["tma", "ldg"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_fused_exchange_across_gpus_bit_exact(cuda_device, world, kernel, tmp_path):
    """Rank r on cuda:r: the fused RS -> Adam -> AG reads every peer's
    gradient shard and writes every peer's parameter chunk over NVLink (TMA
    bulk copies or 128-bit loads / stores of peer memory), bit-exact."""
    _need_gpus(world)
    res = _spawn(world, tmp_path, spread=True, kernel=kernel)
    assert all(str(r["kernel"][0]) == kernel for r in res)
    _check_fused(res, world)


@pytest.mark.parametrize("world", [2, 8])
def test_fused_clipping_across_gpus(cuda_device, world, tmp_path):
    """Global-norm clipping over NVLink: statistics mailboxes on other GPUs."""
    _need_gpus(world)
    max_norm = 0.01
    res = _spawn(world, tmp_path, max_norm, spread=True)
    coefs = [tuple(r["coef"].tolist()) for r in res]
    assert len(set(coefs)) == 1, coefs
    state, norms = _oracle_clipped(world, max_norm, list(coefs[0]))
    for dev_c, want in zip(coefs[0], norms):
        assert want < 1.0 and abs(dev_c - want) <= 1e-6 * want
    for ci in range(len(NUMELS)):
        gathered = ol.allgather([state[ci, r][3] for r in range(world)])
        for r in range(world):
            np.testing.assert_array_equal(res[r][f"master{ci}"].view(np.uint32),
                                          state[ci, r][0].view(np.uint32))
            np.testing.assert_array_equal(res[r][f"param{ci}"], gathered)


def _oracle_clipped(world, max_norm, coefs):
    """Per rank and chunk: (master, gathered params) after STEPS clipped
    steps, each step's clip coefficient taken from the device (checked
    against the oracle's fp64 norm separately)."""
    from paper_2406_08334_b200 import chunks as ch
    state, norms = {}, []
    for step in range(1, STEPS + 1):
        reds, sq = {}, 0.0
        for ci, n in enumerate(NUMELS):
            shard = ol.shard_elems(n, world)
            grads = []
            for q in range(world):
                g = ol.fill_bf16(shard * world, ch.grad_seed(ci, q, step - 1), ch.GRAD_SCALE)
                g[n:] = 0
                grads.append(g)
            for r in range(world):
                red = ol.reduce_scatter(grads, r, shard, fp32=True)
                reds[ci, r] = red
                x = (red * np.float32(1.0 / world)).astype(np.float64)
                sq += float(np.dot(x, x))
        norms.append(min(1.0, max_norm / (np.sqrt(sq) + 1e-6)))
        coef = coefs[step - 1]
        for ci, n in enumerate(NUMELS):
            shard = ol.shard_elems(n, world)
            for r in range(world):
                if (ci, r) not in state:
                    full = ol.fill_f32(shard * world, ch.master_seed(ci), ch.MASTER_SCALE)
                    full[n:] = 0
                    state[ci, r] = [full[r * shard:(r + 1) * shard].copy(),
                                    np.zeros(shard, np.float32), np.zeros(shard, np.float32),
                                    np.zeros(shard, np.uint16)]
                s = ol.scalars(lr=1e-3, weight_decay=0.01, adamw=True, step=step,
                               grad_scale=1.0 / world)
                s.gscale = float(np.float32(s.gscale) * np.float32(coef))
                st = state[ci, r]
                ol.adam_step(s, st[0], st[1], st[2], reds[ci, r], st[3])
    return state, norms


@pytest.mark.parametrize("world", [2, 3])
def test_fused_clipping_across_processes(cuda_device, world, tmp_path):
    """Global-norm clipping in the fused exchange with REAL processes: each
    rank's statistics pass, the 16-byte partials published into every peer's
    mailbox over cudaIpc, rank-order collection (identical coefficient bits
    on every rank), clipped fused update. Bit-exact against the oracle given
    the coefficient; the coefficient within 1e-6 of the oracle's fp64 norm."""
    max_norm = 0.01
    res = _spawn(world, tmp_path, max_norm)
    coefs = [tuple(r["coef"].tolist()) for r in res]
    assert len(set(coefs)) == 1, coefs          # the same bits on every rank, every step
    state, norms = _oracle_clipped(world, max_norm, list(coefs[0]))
    for dev_c, want in zip(coefs[0], norms):
        assert want < 1.0 and abs(dev_c - want) <= 1e-6 * want
    for ci in range(len(NUMELS)):
        params = []
        for r in range(world):
            st = state[ci, r]
            np.testing.assert_array_equal(res[r][f"master{ci}"].view(np.uint32), st[0].view(np.uint32))
            params.append(st[3])
        gathered = ol.allgather(params)
        for r in range(world):
            np.testing.assert_array_equal(res[r][f"param{ci}"], gathered)


def test_bench_self_launch_shared_device_two_ranks(cuda_device):
    """`bench.py --gpus 2` without torchrun re-launches itself with 2 ranks;
    --shared-device puts both on this GPU (cudaIpc peers, fused exchange):
    the N>1 flow end to end, printing one line with n_gpus = 2."""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["PTK_PEER_BARRIER_TIMEOUT_MS"] = "20000"
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2",
                        "--shared-device", "--workload", "flat32", "--steps", "5", "--warmup", "3",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900,
                       env=env, cwd=repo)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["exchange"] == "fused"
    leg = d["exchanges"]["fused"]
    assert leg["consistent_across_ranks"] is True
    assert d["roofline"]["chunks_per_launch"] == 1 and d["e2e"]["value"] > 0


def test_bench_fused_leg_retries_with_register_staged_kernel(cuda_device):
    """At N > 1 the fused exchange runs in a guarded child job; when the
    TMA-ring child fails (here: an injected fault), every rank retries with
    the register-staged kernel and the line records the fallback -- a
    device fault in one kernel cannot lose the N > 1 bench line."""
    import json
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT",
                        "PTK_FUSED_KERNEL")}
    env["PTK_PEER_BARRIER_TIMEOUT_MS"] = "20000"
    env["PTK_BENCH_INJECT_FAULT"] = "fused-tma"
    r = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2",
                        "--shared-device", "--workload", "flat32", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--no-e2e"], capture_output=True, text=True,
                       timeout=600, env=env, cwd=repo)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    leg = json.loads(lines[0])["exchanges"]["fused"]
    assert "TMA-ring fused kernel failed" in leg["fallback"]
    assert "ldg" in leg["kernel"] or "fused_peer_kernel" in leg["kernel"], leg["kernel"]
    assert leg["consistent_across_ranks"] is True
