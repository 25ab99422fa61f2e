"""GPU parity of the chunk step at the BASELINE sizes and of the fused
reduce-scatter -> Adam -> all-gather kernel (virtual ranks on one device).

Full-size checks use size-independent properties: the synthetic inputs are
counter-based (value = f(seed, global index)), so the oracle can recompute any
sampled subset of a 1 GiB chunk exactly and the kernel must match it
bit-for-bit there; padding elements must stay exactly zero.
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle_lib as ol

pytestmark = pytest.mark.gpu


def _modules():
    from paper_2406_08334_b200 import _native, chunks
    return _native, chunks


def _bits(t):
    x = t.cpu().numpy()
    return x.view(np.uint32) if x.dtype == np.float32 else x.view(np.uint16)


def _bf16_bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def _random_numels(seed: int) -> list[int]:
    rng = np.random.default_rng(100 + seed)
    return [int(x) for x in rng.integers(1, 300_000, int(rng.integers(1, 41)))]


@pytest.mark.parametrize("world,numels", [(1, [10_007, 4096]), (2, [10_007, 4096]),
                                          (3, [10_007, 4096]), (4, [10_007, 4096]),
                                          (8, [10_007, 4096]),
                                          # several full TMA tiles per CTA + a partial tile
                                          (2, [2 * 148 * 1024 * 3 + 4104]),
                                          (8, [8 * 148 * 1024 * 2 + 8 * 1000 + 40]),
                                          # seeded random tables of 1-40 ragged chunks
                                          (2, _random_numels(0)), (3, _random_numels(1)),
                                          (5, _random_numels(2)), (8, _random_numels(3))])
def test_fused_virtual_ranks_bit_exact(cuda_device, world, numels):
    """The fused RS -> Adam -> AG kernel (TMA ring by default) over W virtual
    ranks: every rank's fp32 state and every rank's gathered bf16 chunk
    equal the oracle's rank-order fp32 reduce-scatter + Adam + all-gather."""
    nat, ch = _modules()
    sets = [ch.ChunkSet(numels, world=world, rank=r, device=cuda_device, mode="fused")
            for r in range(world)]
    for cs in sets:
        cs.init_synthetic()
        cs.fill_grads(0)
        cs.attach_virtual_peers(sets)
    hyper = ch.AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True)
    # CPU expectation for every rank's shard, from the same counter-based inputs
    for step in (1, 2):
        for cs in sets:
            cs.step(hyper)
        torch.cuda.synchronize()
        # re-fill grads for step 2 so a second RS sees fresh local gradients
        for cs in sets:
            cs.fill_grads(step)
    torch.cuda.synchronize()
    for ci, n in enumerate(numels):
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
            for step in (1, 2):
                grads = []
                for q in range(world):
                    g = ol.fill_bf16(n_pad, ch.grad_seed(ci, q, step - 1), ch.GRAD_SCALE)
                    g[n:] = 0
                    grads.append(g)
                red = ol.reduce_scatter(grads, r, shard, fp32=True)
                ol.adam_step(ol.scalars(lr=1e-3, weight_decay=0.01, adamw=True, step=step,
                                        grad_scale=1.0 / world), mst, m, v, red, out)
            c = sets[r].chunks[ci]
            np.testing.assert_array_equal(_bits(c.master), mst.view(np.uint32))
            np.testing.assert_array_equal(_bits(c.exp_avg), m.view(np.uint32))
            np.testing.assert_array_equal(_bits(c.exp_avg_sq), v.view(np.uint32))
            params.append(out)
        gathered = ol.allgather(params)
        for r in range(world):  # every rank holds the full gathered chunk
            np.testing.assert_array_equal(_bf16_bits(sets[r].chunks[ci].param), gathered)


def test_fused_ldg_variant_bit_exact(cuda_device):
    """The register-staged fused kernel (PTK_FUSED_KERNEL=ldg) passes the same
    oracle checks (the variant is chosen once per process: child pytest)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, PTK_FUSED_KERNEL="ldg")
    r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-q", "-m", "gpu", "-p",
                        "no:cacheprovider", "-k",
                        "fused_virtual_ranks or fused_global_norm or fused_nonfinite"],
                       env=env, capture_output=True, text=True, timeout=900,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    # 16 small-size cases + the 4 full-size cfg2 cases of the fused exchange
    assert "20 passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:]


def _fused_sets(ch, numels, world, dev):
    sets = [ch.ChunkSet(numels, world=world, rank=r, device=dev, mode="fused")
            for r in range(world)]
    for cs in sets:
        cs.init_synthetic()
        cs.fill_grads(0)
        cs.attach_virtual_peers(sets)
    return sets


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_fused_global_norm_clipping_virtual_ranks(cuda_device, world):
    """Clipping in the fused exchange: statistics pass over every rank's
    reduced gradient shards (ptk_fused_grad_stats_table), 16-byte partials
    exchanged through the peer mailboxes (rank-order sum: the same bits on
    every rank), device clip coefficient read by the fused update. Checked
    against the oracle's fp64 global norm (1e-6) and, given the device
    coefficient, bit-exactly on every rank's state and gathered chunk."""
    nat, ch = _modules()
    numels = [10_007, 3 * 4096 + 8]
    sets = _fused_sets(ch, numels, world, cuda_device)
    hyper = ch.AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True)
    max_norm = 0.01
    ch.fused_group_step(sets, hyper, max_grad_norm=max_norm)
    torch.cuda.synchronize()
    coefs = [float(cs.clip_coef[0]) for cs in sets]
    assert len(set(coefs)) == 1, coefs                 # identical on every rank
    assert len({tuple(cs.stats.cpu().tolist()) for cs in sets}) == 1
    coef = coefs[0]
    sq = 0.0
    reduced = {}
    for ci, n in enumerate(numels):
        shard = ol.shard_elems(n, world)
        grads = []
        for q in range(world):
            g = ol.fill_bf16(shard * world, ch.grad_seed(ci, q, 0), ch.GRAD_SCALE)
            g[n:] = 0
            grads.append(g)
        for r in range(world):
            red = ol.reduce_scatter(grads, r, shard, fp32=True)
            reduced[ci, r] = red
            scaled = (red * np.float32(1.0 / world)).astype(np.float64)
            sq += float(np.dot(scaled, scaled))
    want = min(1.0, max_norm / (np.sqrt(sq) + 1e-6))
    assert want < 1.0 and abs(coef - want) <= 1e-6 * want
    assert abs(float(sets[0].stats[0]) - sq) <= 1e-6 * sq
    for ci, n in enumerate(numels):
        shard = ol.shard_elems(n, world)
        master_full = ol.fill_f32(shard * world, ch.master_seed(ci), ch.MASTER_SCALE)
        master_full[n:] = 0
        params = []
        for r in range(world):
            mst = master_full[r * shard:(r + 1) * shard].copy()
            m = np.zeros(shard, np.float32)
            v = np.zeros(shard, np.float32)
            out = np.zeros(shard, np.uint16)
            s = ol.scalars(lr=1e-3, weight_decay=0.01, adamw=True, step=1, grad_scale=1.0 / world)
            s.gscale = float(np.float32(s.gscale) * np.float32(coef))
            ol.adam_step(s, mst, m, v, reduced[ci, r], out)
            c = sets[r].chunks[ci]
            np.testing.assert_array_equal(_bits(c.master), mst.view(np.uint32))
            np.testing.assert_array_equal(_bits(c.exp_avg_sq), v.view(np.uint32))
            params.append(out)
        gathered = ol.allgather(params)
        for r in range(world):
            np.testing.assert_array_equal(_bf16_bits(sets[r].chunks[ci].param), gathered)
    # a second clipped step uses fresh epochs of the same mailboxes
    for cs in sets:
        cs.fill_grads(1)
    ch.fused_group_step(sets, hyper, max_grad_norm=max_norm)
    torch.cuda.synchronize()
    assert len({float(cs.clip_coef[0]) for cs in sets}) == 1


def test_fused_nonfinite_skips_every_rank(cuda_device):
    """One rank's non-finite gradient element skips the step on ALL ranks
    (global overflow flag from the mailbox exchange): no state or parameter
    changes anywhere."""
    nat, ch = _modules()
    world = 4
    sets = _fused_sets(ch, [4096, 8200], world, cuda_device)
    sets[2].chunks[1].grad[100] = float("inf")
    before = [[(c.master.clone(), c.param.clone()) for c in cs.chunks] for cs in sets]
    ch.fused_group_step(sets, ch.AdamHyper(), skip_nonfinite=True)
    torch.cuda.synchronize()
    for cs, b in zip(sets, before):
        assert int(cs.skip_flag[0]) == 1
        assert int(cs.stats.view(torch.int64)[1]) == 1
        for (m0, p0), c in zip(b, cs.chunks):
            assert torch.equal(m0, c.master) and torch.equal(p0, c.param)


def _world1_comm(nat):
    """A real NCCL communicator of one rank: RS / AG / stats all-reduce then
    go through NCCL (in place, a local copy) exactly as at w > 1."""
    uid = (ctypes.c_uint8 * nat.PTK_UNIQUE_ID_BYTES)()
    nat.lib.ptk_comm_unique_id(uid)
    comm = ctypes.c_void_p()
    nat.lib.ptk_comm_init(ctypes.byref(comm), 1, 0, uid)
    return comm


@pytest.mark.parametrize("with_comm,symmetric", [(False, False), (True, False), (True, True)])
def test_nccl_mode_single_rank_matches_oracle(cuda_device, with_comm, symmetric):
    """symmetric: the chunk buffers are ncclMemAlloc'd and registered as NCCL
    symmetric windows (the NCCL baseline's strongest path); same bits."""
    nat, ch = _modules()
    numels = [123_457, 65_536]
    comm = _world1_comm(nat) if with_comm else None
    cs = ch.ChunkSet(numels, world=1, rank=0, device=cuda_device, mode="nccl", comm=comm,
                     symmetric=symmetric)
    if symmetric:
        assert len(cs._windows) == 2 * len(numels)
    cs.init_synthetic()
    cs.fill_grads(0)
    hyper = ch.AdamHyper()
    for _ in range(3):
        cs.step(hyper)
    torch.cuda.synchronize()
    for ci, n in enumerate(numels):
        c = cs.chunks[ci]
        mst = ol.fill_f32(c.shard, ch.master_seed(ci), ch.MASTER_SCALE)
        mst[n:] = 0
        g = ol.fill_bf16(c.shard, ch.grad_seed(ci, 0, 0), ch.GRAD_SCALE)
        g[n:] = 0
        m = np.zeros(c.shard, np.float32)
        v = np.zeros(c.shard, np.float32)
        out = np.zeros(c.shard, np.uint16)
        for step in (1, 2, 3):
            ol.adam_step(ol.scalars(step=step), mst, m, v, g, out)
        np.testing.assert_array_equal(_bits(c.master), mst.view(np.uint32))
        np.testing.assert_array_equal(_bf16_bits(c.param), out)
    if comm is not None:
        # clipping path: RS -> stats -> NCCL stats all-reduce -> clip -> Adam -> AG
        cs.step(ch.AdamHyper(), max_grad_norm=1.0, skip_nonfinite=True)
        torch.cuda.synchronize()
        assert cs.grad_stats()[1] == 0
        nat.lib.ptk_comm_barrier(comm, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        cs.close()   # deregisters the symmetric windows (collective) before the comm goes
        assert cs._windows == []
        nat.lib.ptk_comm_destroy(comm)


def test_cuda_graph_of_steps_matches_eager(cuda_device):
    """bench.py times the K steps as ONE replay of a CUDA graph holding them
    (each step captured with its own step number). That replay must leave
    exactly the state of K host-launched steps: master / m / v / params bit
    for bit, and the last step's gradient statistics."""
    nat, ch = _modules()
    numels = [1_000_003, 3 * 1536 * 148 + 77]   # partial tile + several full waves

    def make():
        cs = ch.ChunkSet(numels, device=cuda_device)
        cs.init_synthetic()
        cs.fill_grads(0)
        return cs

    hyper = ch.AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True)
    eager, graphed = make(), make()
    for _ in range(4):
        eager.step(hyper)
    launches0 = nat.launch_count()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(4):
            graphed.step(hyper)
    captured = nat.launch_count() - launches0
    torch.cuda.synchronize()
    # capture performs no work: the state is still the initial one
    assert torch.equal(graphed.chunks[0].exp_avg, torch.zeros_like(graphed.chunks[0].exp_avg))
    g.replay()
    torch.cuda.synchronize()
    assert captured == 4 * 2   # per step: stats reset + ONE chunk-table Adam launch
    for a, b in zip(eager.chunks, graphed.chunks):
        for x, y in ((a.master, b.master), (a.exp_avg, b.exp_avg), (a.exp_avg_sq, b.exp_avg_sq),
                     (a.param, b.param)):
            assert torch.equal(x.view(torch.int32) if x.dtype == torch.float32 else
                               x.view(torch.int16),
                               y.view(torch.int32) if y.dtype == torch.float32 else
                               y.view(torch.int16))
    assert eager.grad_stats() == graphed.grad_stats()


def test_multi_rank_nccl_needs_a_communicator(cuda_device):
    _, ch = _modules()
    with pytest.raises(ValueError, match="communicator"):
        ch.ChunkSet([1024], world=2, rank=0, device=cuda_device, mode="nccl")


FULL_SIZE = {  # workload -> (parameters, chunks): SURVEY §8(a) golden layouts
    "gpt2-1b_b2": (985_376_256, 4),
    "gpt2-1.5b_b8": (1_557_608_000, 3),
    "gpt2-10b_b8": (9_876_279_296, 49),   # 158 GB of chunk state on one B200
    "flat512": (268_435_456, 1),           # one flat 512 MiB chunk (cfg5's largest point)
    # maximum size: one chunk of 2^31 + 4101 parameters (element offsets beyond
    # int32, fp32 state beyond 2^33 bytes, a ragged count padded to 8)
    "flat_2g": (2_147_487_749, 1),
}
PARITY_STEPS = 10  # 10 steps, fresh gradients (seed 1 + rank + step) each step
HYPERS = {"adam": dict(), "adamw_wd0.01": dict(weight_decay=0.01, adamw=True)}


def _sample_fill(fill, n_idx, seed, scale, idx):
    return np.array([fill(1, seed, scale, int(i))[0] for i in idx],
                    np.float32 if fill is ol.fill_f32 else np.uint16)


@pytest.mark.parametrize("variant", sorted(HYPERS))
@pytest.mark.parametrize("workload", sorted(FULL_SIZE))
def test_full_size_layout_sampled_parity(cuda_device, workload, variant):
    """cfg1 / cfg2 / cfg3 / flat 512 MiB / one 2^31+ element chunk at full size on one GPU (cfg3: 49
    chunks, 9.9 B params, fp32 master/m/v + bf16 param/grad = 158 GB
    resident): 10 steps with FRESH gradients every step (Adam, and AdamW
    with weight decay 0.01), then sampled elements (head, tail, random) of
    every chunk are recomputed by the oracle from their global index over the
    same 10 steps and must match bit-exactly (master, m, v, bf16 param);
    the last step's statistics must equal the full-chunk sum of squares
    within 1e-6 (the oracle's on the host up to 2 B params, torch fp64 on the
    device above); padding elements stay exactly zero."""
    nat, ch = _modules()
    if workload.startswith("flat"):
        numels = [FULL_SIZE[workload][0]]
    else:
        from paper_2406_08334_b200 import planner
        layout = planner.layout_for(workload)
        numels = [c["used_bytes"] // layout["bytes_per_param"] for c in layout["chunks"]]
    assert (sum(numels), len(numels)) == FULL_SIZE[workload]
    host_sum = sum(numels) <= 2_000_000_000
    cs = ch.ChunkSet(numels, world=1, rank=0, device=cuda_device)
    cs.init_synthetic()
    hyper = ch.AdamHyper(**HYPERS[variant])
    for step in range(1, PARITY_STEPS + 1):
        cs.fill_grads(step - 1)
        cs.step(hyper)
    torch.cuda.synchronize()
    sumsq, bad = cs.grad_stats()
    assert bad == 0
    rng = np.random.default_rng(0)
    total_sq = 0.0
    last = PARITY_STEPS - 1
    for ci, n in enumerate(numels):
        c = cs.chunks[ci]
        idx = np.unique(np.concatenate([np.arange(0, 64), np.arange(n - 64, n),
                                        rng.integers(0, n, 2048 if host_sum else 256)]))
        mst = _sample_fill(ol.fill_f32, idx.size, ch.master_seed(ci), ch.MASTER_SCALE, idx)
        m = np.zeros(idx.size, np.float32)
        v = np.zeros(idx.size, np.float32)
        out = np.zeros(idx.size, np.uint16)
        for step in range(1, PARITY_STEPS + 1):
            g = _sample_fill(ol.fill_bf16, idx.size, ch.grad_seed(ci, 0, step - 1),
                             ch.GRAD_SCALE, idx)
            ol.adam_step(ol.scalars(step=step, **HYPERS[variant]), mst, m, v, g, out)
        ti = torch.from_numpy(idx).to(cuda_device)
        np.testing.assert_array_equal(_bits(c.master[ti]), mst.view(np.uint32))
        np.testing.assert_array_equal(_bits(c.exp_avg[ti]), m.view(np.uint32))
        np.testing.assert_array_equal(_bits(c.exp_avg_sq[ti]), v.view(np.uint32))
        np.testing.assert_array_equal(_bf16_bits(c.param[ti]), out)
        # full-chunk grad statistics of the last step
        if host_sum:
            gf = ol.bf16_to_f32(ol.fill_bf16(n, ch.grad_seed(ci, 0, last), ch.GRAD_SCALE))
            total_sq += float(np.dot(gf.astype(np.float64), gf.astype(np.float64)))
        else:
            for lo in range(0, n, 1 << 27):
                gd = c.grad[lo:min(n, lo + (1 << 27))].double()
                total_sq += float(torch.dot(gd, gd))
            del gd
        if c.n_pad > n:
            assert torch.count_nonzero(c.param[n:]).item() == 0
            assert torch.count_nonzero(c.master[n:]).item() == 0
    assert abs(sumsq - total_sq) <= 1e-6 * total_sq


@pytest.mark.parametrize("variant", sorted(HYPERS))
@pytest.mark.parametrize("world", [2, 8])
def test_full_size_fused_virtual_ranks_sampled_parity(cuda_device, world, variant):
    """cfg2 (GPT-2 1.5B, 3 x 1 GiB chunks) at full size through the fused
    RS -> Adam -> AG exchange over W virtual ranks on this device (W = 8:
    8 ranks' bf16 param + grad chunks and the sharded fp32 state, 68 GB):
    10 steps with FRESH gradients on every rank every step (Adam, and AdamW
    with weight decay 0.01); then sampled elements (head, tail, every shard
    boundary, random) are recomputed by the oracle from their global index
    -- rank-order fp32 sum of the W ranks' bf16 gradients, Adam with grad
    scale 1/W -- and must match bit-exactly in the owner's master / m / v
    and in EVERY rank's gathered bf16 chunk."""
    nat, ch = _modules()
    from paper_2406_08334_b200 import planner
    layout = planner.layout_for("gpt2-1.5b_b8")
    numels = [c["used_bytes"] // layout["bytes_per_param"] for c in layout["chunks"]]
    sets = [ch.ChunkSet(numels, world=world, rank=r, device=cuda_device, mode="fused")
            for r in range(world)]
    for cs in sets:
        cs.init_synthetic()
        cs.attach_virtual_peers(sets)
    hyper = ch.AdamHyper(**HYPERS[variant])
    for step in range(1, PARITY_STEPS + 1):
        for cs in sets:
            cs.fill_grads(step - 1)
        ch.fused_group_step(sets, hyper)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    for ci, n in enumerate(numels):
        shard = sets[0].chunks[ci].shard
        bounds = np.concatenate([np.arange(r * shard - 4, r * shard + 4) for r in range(1, world)])
        idx = np.unique(np.concatenate([np.arange(0, 32), np.arange(n - 32, n), bounds,
                                        rng.integers(0, n, 384)]))
        mst = _sample_fill(ol.fill_f32, idx.size, ch.master_seed(ci), ch.MASTER_SCALE, idx)
        m = np.zeros(idx.size, np.float32)
        v = np.zeros(idx.size, np.float32)
        out = np.zeros(idx.size, np.uint16)
        for step in range(1, PARITY_STEPS + 1):
            grads = [_sample_fill(ol.fill_bf16, idx.size, ch.grad_seed(ci, q, step - 1),
                                  ch.GRAD_SCALE, idx) for q in range(world)]
            red = ol.reduce_scatter(grads, 0, idx.size, fp32=True)   # rank-order fp32 sum
            ol.adam_step(ol.scalars(step=step, grad_scale=1.0 / world, **HYPERS[variant]),
                         mst, m, v, red, out)
        owner = idx // shard
        for r in range(world):
            mine = owner == r
            if mine.any():
                c = sets[r].chunks[ci]
                ti = torch.from_numpy(idx[mine] - r * shard).to(cuda_device)
                np.testing.assert_array_equal(_bits(c.master[ti]), mst[mine].view(np.uint32))
                np.testing.assert_array_equal(_bits(c.exp_avg[ti]), m[mine].view(np.uint32))
                np.testing.assert_array_equal(_bits(c.exp_avg_sq[ti]), v[mine].view(np.uint32))
            tg = torch.from_numpy(idx).to(cuda_device)
            np.testing.assert_array_equal(_bf16_bits(sets[r].chunks[ci].param[tg]), out)
    for cs in sets:
        cs.close()


def test_global_norm_clipping_matches_oracle(cuda_device):
    """max_grad_norm: global norm over all chunks -> device clip coefficient ->
    every chunk's Adam reads it from device memory. Checked against the
    oracle with the same coefficient (bit-exact state) and the coefficient
    against the oracle's fp64 norm."""
    nat, ch = _modules()
    numels = [50_001, 70_003]
    cs = ch.ChunkSet(numels, world=1, rank=0, device=cuda_device)
    cs.init_synthetic()
    cs.fill_grads(0)
    max_norm = 0.05
    cs.step(ch.AdamHyper(), max_grad_norm=max_norm)
    torch.cuda.synchronize()
    coef = float(cs.clip_coef[0])
    sq = 0.0
    for ci, n in enumerate(numels):
        g = ol.bf16_to_f32(ol.fill_bf16(n, ch.grad_seed(ci, 0, 0), ch.GRAD_SCALE))
        sq += float(np.dot(g.astype(np.float64), g.astype(np.float64)))
    want = min(1.0, max_norm / (np.sqrt(sq) + 1e-6))
    assert want < 1.0 and abs(coef - want) <= 1e-6 * want
    for ci, n in enumerate(numels):
        c = cs.chunks[ci]
        mst = ol.fill_f32(c.shard, ch.master_seed(ci), ch.MASTER_SCALE)
        mst[n:] = 0
        g = ol.fill_bf16(c.shard, ch.grad_seed(ci, 0, 0), ch.GRAD_SCALE)
        g[n:] = 0
        s = ol.scalars(step=1)
        s.gscale = float(np.float32(s.gscale) * np.float32(coef))
        m = np.zeros(c.shard, np.float32)
        v = np.zeros(c.shard, np.float32)
        out = np.zeros(c.shard, np.uint16)
        ol.adam_step(s, mst, m, v, g, out)
        np.testing.assert_array_equal(_bits(c.master), mst.view(np.uint32))
        np.testing.assert_array_equal(_bf16_bits(c.param), out)


def test_nonfinite_gradient_skips_the_whole_step(cuda_device):
    nat, ch = _modules()
    cs = ch.ChunkSet([4096, 8192], world=1, rank=0, device=cuda_device)
    cs.init_synthetic()
    cs.fill_grads(0)
    cs.chunks[1].grad[100] = float("inf")
    before = [c.master.clone() for c in cs.chunks]
    cs.step(ch.AdamHyper(), skip_nonfinite=True)
    torch.cuda.synchronize()
    assert int(cs.skip_flag[0]) == 1
    for b, c in zip(before, cs.chunks):
        assert torch.equal(b, c.master)  # no chunk updated, not even the finite one


def test_pinned_copies_round_trip(cuda_device):
    nat, ch = _modules()
    n = 1 << 20
    host = ctypes.c_void_p()
    nat.lib.ptk_host_alloc_pinned(ctypes.byref(host), 2 * n)
    src = torch.arange(n, dtype=torch.int16)
    ctypes.memmove(host, src.data_ptr(), 2 * n)
    dev = torch.zeros(n, dtype=torch.int16, device=cuda_device)
    s = ctypes.c_void_p()
    nat.lib.ptk_stream_create(ctypes.byref(s), 1)
    nat.lib.ptk_memcpy_h2d_async(ctypes.c_void_p(dev.data_ptr()), host, 2 * n, s)
    nat.lib.ptk_stream_synchronize(s)
    assert torch.equal(dev.cpu(), src)
    dev.mul_(2)
    torch.cuda.synchronize()
    nat.lib.ptk_memcpy_d2h_async(host, ctypes.c_void_p(dev.data_ptr()), 2 * n, s)
    nat.lib.ptk_stream_synchronize(s)
    back = torch.empty(n, dtype=torch.int16)
    ctypes.memmove(back.data_ptr(), host, 2 * n)
    assert torch.equal(back, src * 2)
    nat.lib.ptk_stream_destroy(s)
    nat.lib.ptk_host_free_pinned(host)


@pytest.mark.parametrize("world,shard", [(1, 4101), (2, 2048 * 150 + 8), (3, 1000),
                                         (8, 8 * 1024 + 8)])
def test_peer_reduce_scatter_and_allgather_match_oracle(cuda_device, world, shard):
    """The non-persistent chunks' peer exchange over W virtual ranks' buffers:
    ptk_peer_reduce_scatter_f32 = the oracle's rank-order fp32 reduce-scatter
    bit for bit (every rank's shard; W = 1 with an unpadded n % 8 tail), and
    ptk_peer_allgather assembles every rank's shard into each rank's buffer."""
    nat, ch = _modules()
    n_pad = world * shard
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    host = [ol.fill_bf16(n_pad, 70 + r, ch.GRAD_SCALE) for r in range(world)]
    dev = [torch.from_numpy(h.view(np.int16).copy()).to(cuda_device) for h in host]
    ptrs = (ctypes.c_void_p * nat.PTK_MAX_PEERS)(*[t.data_ptr() for t in dev])
    for r in range(world):
        out = torch.empty(shard, dtype=torch.float32, device=cuda_device)
        nat.lib.ptk_peer_reduce_scatter_f32(ptrs, world, r, shard, ch.vp(out), s)
        want = ol.reduce_scatter(host, r, shard, fp32=True)
        np.testing.assert_array_equal(_bits(out), want.view(np.uint32))
    # all-gather: each rank's buffer holds only its own shard, then pulls the rest
    bufs = [torch.zeros(n_pad, dtype=torch.int16, device=cuda_device) for _ in range(world)]
    for r, b in enumerate(bufs):
        b[r * shard:(r + 1) * shard] = dev[r][r * shard:(r + 1) * shard]
    bp = (ctypes.c_void_p * nat.PTK_MAX_PEERS)(*[b.data_ptr() for b in bufs])
    for r in range(world):
        nat.lib.ptk_peer_allgather(bp, world, r, 2 * shard, s)
    torch.cuda.synchronize()
    want = ol.allgather([h[r * shard:(r + 1) * shard] for r, h in enumerate(host)])
    for b in bufs:
        np.testing.assert_array_equal(b.cpu().numpy().view(np.uint16), want)
