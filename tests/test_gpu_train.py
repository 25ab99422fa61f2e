"""End-to-end: a GPT-2 shaped model whose parameters live in the planner's
chunk buffers trains through the chunk data plane exactly like a plain PyTorch
model trained with torch.optim.AdamW on fp32 master weights.

Reference: the same operator sequence on ordinary bf16 leaf tensors, grads
cast to fp32, torch.optim.AdamW(foreach=False) on fp32 masters, bf16 copy-back.
Step-1 loss must be bit-identical (same bf16 weights, same kernels); the loss
trajectory over 6 steps within 2e-3 relative, and the fp32 masters within the
oracle-vs-torch Adam tolerance (the chunk Adam follows torch's update order
without FMA contraction, tests/test_oracle.py).
"""
import json
import os
import types

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(tmp_path, cuda_device):
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import ChunkSet
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps({"hidden_size": 256, "n_blocks": 2, "n_heads": 4,
                                "vocab_size": 1000, "seq_len": 128}))
    tpath = planner.trace_file(["--spec", str(spec), "--batch", "4"], str(tmp_path / "t.json"))
    trace = json.load(open(tpath))
    layout = planner.pack(tpath, grid="2Mi")
    assert len(layout["chunks"]) == 3  # embedding | block 0 | block 1 (+ head, loss)
    numels = [c["used_bytes"] // 2 for c in layout["chunks"]]
    cs = ChunkSet(numels, world=1, rank=0, device=cuda_device)
    shape = GPT2Shape.from_trace_meta(trace["meta"], trace["n_blocks"])
    model = ChunkedGPT2(shape, layout, cs, trace["ops"])
    model.init_weights(seed=0)
    return model, shape


def test_chunked_training_matches_plain_torch(tmp_path, cuda_device):
    from paper_2406_08334_b200.chunks import AdamHyper
    from paper_2406_08334_b200.train import ChunkedGPT2, train_step
    model, shape = _setup(tmp_path, cuda_device)
    # plain-PyTorch twin with copies of the initial weights
    def clone(d):
        return {k: v.detach().clone().requires_grad_(True) for k, v in d.items()}
    twin = types.SimpleNamespace(shape=shape, params=clone(model.params),
                                 blocks=[clone(b) for b in model.blocks])
    leaves = list(twin.params.values()) + [p for b in twin.blocks for p in b.values()]
    masters = [p.detach().float().clone().requires_grad_(True) for p in leaves]
    opt = torch.optim.AdamW(masters, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.01,
                            foreach=False)
    hyper = AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True)
    g = torch.Generator(device=cuda_device).manual_seed(0)
    views = list(model.params.values()) + [p for b in model.blocks for p in b.values()]

    def check_masters(rtol, atol):
        # fp32 masters vs torch's AdamW masters, parameter by parameter
        for v, m in zip(views, masters):
            c = next(c for c in model.chunks.chunks
                     if c.param.data_ptr() <= v.data_ptr() < c.param.data_ptr() + 2 * c.n_pad)
            lo = (v.data_ptr() - c.param.data_ptr()) // 2
            np.testing.assert_allclose(c.master[lo:lo + v.numel()].cpu().numpy(),
                                       m.detach().flatten().cpu().numpy(), rtol=rtol, atol=atol)

    ours, ref = [], []
    for step in range(6):
        # learnable synthetic data: the next token is the current one + 1
        x = torch.randint(0, shape.vocab, (4, shape.seq), device=cuda_device, generator=g)
        y = (x + 1) % shape.vocab
        ours.append(float(train_step(model, x, y, hyper)))
        loss = ChunkedGPT2.loss(twin, x, y)
        loss.backward()
        for mp, p in zip(masters, leaves):
            mp.grad = p.grad.float()
            p.grad = None
        opt.step()
        with torch.no_grad():
            for mp, p in zip(masters, leaves):
                p.copy_(mp)
        ref.append(float(loss.detach()))
        if step == 0:
            # identical inputs and gradients: the update agrees to fp32 rounding
            # (same rule as torch; torch's CPU/GPU kernels may fuse, ours never do)
            check_masters(rtol=1e-5, atol=1e-8)
    assert ours[0] == ref[0]
    # afterwards the trajectories stay together in loss (elements whose
    # gradient is ~0 flip sign under Adam's normalisation, so per-element
    # masters are not comparable after the first step)
    np.testing.assert_allclose(ours, ref, rtol=2e-3)
    assert ours[-1] < ours[0]


@pytest.mark.parametrize("schedule", [["swap", "checkpoint"], ["checkpoint", "swap"],
                                      ["swap", "swap"]])
def test_block_schedule_swap_checkpoint_is_exact(tmp_path, cuda_device, schedule):
    """Swap (activations to pinned host on a side stream) and checkpoint
    (recompute) change where activations live, never the numbers: the loss
    trajectory and the updated chunk state are bit-identical to keeping
    everything resident."""
    from paper_2406_08334_b200.chunks import AdamHyper
    from paper_2406_08334_b200.train import train_step
    runs = []
    for sched in (["none", "none"], schedule):
        model, shape = _setup(_fresh(tmp_path, "_".join(sched)), cuda_device)
        model.set_block_schedule(sched)
        g = torch.Generator(device=cuda_device).manual_seed(0)
        hyper = AdamHyper(lr=1e-3)
        losses = []
        for _ in range(3):
            x = torch.randint(0, shape.vocab, (4, shape.seq), device=cuda_device, generator=g)
            losses.append(float(train_step(model, x, (x + 1) % shape.vocab, hyper)))
        torch.cuda.synchronize()
        runs.append((losses, torch.cat([c.master for c in model.chunks.chunks]).cpu()))
    assert runs[0][0] == runs[1][0]
    assert torch.equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("n_persist,n_buffer,schedule", [
    (1, 1, None), (0, 2, None), (1, 2, None),
    (0, 1, ["checkpoint", "swap"]), (1, 1, ["swap", "checkpoint"]), (0, 2, ["checkpoint", "checkpoint"])])
def test_non_persistent_chunks_train_bit_identically(tmp_path, cuda_device, n_persist, n_buffer,
                                                     schedule):
    """ZeRO-offload inside the training model: non-persistent chunks live in
    pinned host memory, are fetched into n_buffer device slots before use
    (re-gathered in backward when evicted), their gradients are offloaded and
    updated by the host Adam. Because the host Adam is bit-identical to the
    device Adam, the loss trajectory and every master weight must equal the
    all-persistent run exactly."""
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.offload import ChunkPool
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, train_step

    def run(np_, nb, sched=None):
        d = _fresh(tmp_path, f"np{np_}nb{nb}{sched}")
        spec = d / "spec.json"
        spec.write_text(json.dumps({"hidden_size": 256, "n_blocks": 2, "n_heads": 4,
                                    "vocab_size": 1000, "seq_len": 128}))
        tpath = planner.trace_file(["--spec", str(spec), "--batch", "4"], str(d / "t.json"))
        trace = json.load(open(tpath))
        layout = planner.pack(tpath, grid="2Mi")
        numels = [c["used_bytes"] // 2 for c in layout["chunks"]]
        cs = ChunkSet(numels[:np_], device=cuda_device)
        # small ragged pieces: D2H -> host Adam -> H2D pipelined within a chunk
        pool = (ChunkPool(numels, np_, nb, device=cuda_device, piece=65_544)
                if np_ < len(numels) else None)
        shape = GPT2Shape.from_trace_meta(trace["meta"], trace["n_blocks"])
        model = ChunkedGPT2(shape, layout, cs, trace["ops"], pool=pool)
        model.init_weights(seed=0)
        if sched:
            model.set_block_schedule(sched)
        g = torch.Generator(device=cuda_device).manual_seed(0)
        losses = []
        for _ in range(4):
            x = torch.randint(0, shape.vocab, (4, shape.seq), device=cuda_device, generator=g)
            losses.append(float(train_step(model, x, (x + 1) % shape.vocab,
                                           AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True))))
        torch.cuda.synchronize()
        masters = [c.master.cpu() for c in cs.chunks]
        if pool is not None:
            pool.finish_step()
            masters += [pool.h_master[c][:pool.numel[c]].clone() for c in sorted(pool.numel)]
            counters = dict(pool.counters)
        else:
            counters = {}
        return losses, [m[:n] for m, n in zip(masters, numels)], counters

    ref_losses, ref_masters, _ = run(3, 0)
    losses, masters, counters = run(n_persist, n_buffer, schedule)
    assert losses == ref_losses
    for a, b in zip(masters, ref_masters):
        assert torch.equal(a, b)
    pooled = 3 - n_persist
    assert counters["fetch"] >= 4 * pooled          # at least one fetch per chunk per step
    assert counters["d2h_bytes"] > 0 and counters["h2d_bytes"] > 0


LLAMA_SPEC = {"hidden_size": 256, "n_blocks": 2, "n_heads": 4, "n_kv_heads": 2, "ffn_hidden": 688,
              "vocab_size": 1000, "seq_len": 128, "gated_mlp": True, "bias": False,
              "tied_embeddings": False, "learned_pos_embedding": False}


def test_llama_shape_trains_and_offloads_bit_identically(tmp_path, cuda_device):
    """The Llama family (RMSNorm, rotary, grouped KV, SwiGLU, untied head):
    the architecture is recovered from the trace's parameter bytes, trains,
    and with every chunk non-persistent (host Adam, 2 device buffers) gives
    the all-persistent run's losses and masters bit for bit."""
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.offload import ChunkPool
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, train_step

    spec = tmp_path / "llama.json"
    spec.write_text(json.dumps(LLAMA_SPEC))
    tpath = planner.trace_file(["--spec", str(spec), "--batch", "4"], str(tmp_path / "t.json"))
    trace = json.load(open(tpath))
    layout = planner.pack(tpath, grid="2Mi")
    numels = [c["used_bytes"] // 2 for c in layout["chunks"]]
    shape = GPT2Shape.from_trace(trace)
    assert shape.gated and not shape.bias and not shape.tied and shape.kv_heads == 2

    def run(np_, nb):
        cs = ChunkSet(numels[:np_], device=cuda_device)
        pool = ChunkPool(numels, np_, nb, device=cuda_device) if np_ < len(numels) else None
        model = ChunkedGPT2(shape, layout, cs, trace["ops"], pool=pool)
        model.init_weights(seed=0)
        g = torch.Generator(device=cuda_device).manual_seed(0)
        losses = []
        for _ in range(4):
            x = torch.randint(0, shape.vocab, (4, shape.seq), device=cuda_device, generator=g)
            losses.append(float(train_step(model, x, (x + 1) % shape.vocab, AdamHyper(lr=1e-3))))
        torch.cuda.synchronize()
        ms = [c.master.cpu() for c in cs.chunks]
        if pool is not None:
            pool.finish_step()
            ms += [pool.h_master[c].clone() for c in sorted(pool.numel)]
        return losses, [m[:n] for m, n in zip(ms, numels)]

    ref_l, ref_m = run(len(numels), 0)
    l, m = run(0, 2)
    assert l == ref_l and ref_l[-1] < ref_l[0]
    for a, b in zip(m, ref_m):
        assert torch.equal(a, b)


def test_profiler_measures_a_loadable_trace(tmp_path, cuda_device):
    """The profiler's measured trace has the synthesized trace's operators and
    parameter bytes, positive measured times that add up to the measured
    iteration, retained activations, and loads into the planner unchanged."""
    import subprocess
    from paper_2406_08334_b200.profiler import profile_trace
    model, shape = _setup(tmp_path, cuda_device)
    x = torch.randint(0, shape.vocab, (4, shape.seq), device=cuda_device)
    measured = profile_trace(model, x, (x + 1) % shape.vocab, reps=2)
    synth = json.load(open(tmp_path / "t.json"))
    assert [o["name"] for o in measured["ops"]] == [o["name"] for o in synth["ops"]]
    assert [o["param_bytes"] for o in measured["ops"]] == [o["param_bytes"] for o in synth["ops"]]
    assert all(o["t_fwd"] > 0 for o in measured["ops"])
    assert sum(o["t_bwd"] for o in measured["ops"]) > 0
    assert sum(o["act_bytes"] for o in measured["ops"]) > 0
    path = tmp_path / "measured.json"
    path.write_text(json.dumps(measured))
    memplan = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "build", "memplan")
    out = subprocess.run([memplan, "pack", "--trace", str(path), "--grid", "2Mi"], check=True,
                         capture_output=True, text=True).stdout
    assert json.loads(out)["n_chunk"] == 3


def _fresh(tmp_path, name):
    d = tmp_path / name
    d.mkdir(parents=True, exist_ok=True)
    return d


def test_chunked_parameters_are_chunk_views(tmp_path, cuda_device):
    model, shape = _setup(tmp_path, cuda_device)
    c0 = model.chunks.chunks[0]
    wte = model.params["wte"]
    assert wte.data_ptr() == c0.param.data_ptr()  # op 0 starts chunk 0
    wpe = model.params["wpe"]
    assert wpe.data_ptr() == c0.param.data_ptr() + 2 * wte.numel()
    blk1 = model.chunks.chunks[2]
    assert model.blocks[1]["ln1_w"].data_ptr() == blk1.param.data_ptr()


def test_training_timeline_in_simulator_schema(tmp_path, cuda_device):
    """The measured timeline of one training iteration (paper_2406_08334_b200
    .timeline) has the simulator's schema: per block fwd/bwd start/end in
    order, one upload / offload / host update per pooled chunk, one device
    optim per persistent chunk; the CSV round-trips and summarises."""
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.offload import ChunkPool
    from paper_2406_08334_b200.timeline import Timeline, read_csv, summarize, write_csv
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, train_step
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps({"hidden_size": 256, "n_blocks": 2, "n_heads": 4,
                                "vocab_size": 1000, "seq_len": 128}))
    tpath = planner.trace_file(["--spec", str(spec), "--batch", "4"], str(tmp_path / "t.json"))
    trace = json.load(open(tpath))
    layout = planner.pack(tpath, grid="2Mi")
    numels = [c["used_bytes"] // 2 for c in layout["chunks"]]
    cs = ChunkSet(numels[:1], device=cuda_device)
    pool = ChunkPool(numels, 1, 1, device=cuda_device)
    model = ChunkedGPT2(GPT2Shape.from_trace(trace), layout, cs, trace["ops"], pool=pool)
    model.init_weights(0)
    model.set_block_schedule(["checkpoint", "swap"])
    x = torch.randint(0, 1000, (4, 128), device=cuda_device)
    for _ in range(2):
        train_step(model, x, (x + 1) % 1000, AdamHyper())
    pool.finish_step()
    tl = Timeline()
    model.timeline = cs.timeline = pool.timeline = tl
    tl.begin()
    train_step(model, x, (x + 1) % 1000, AdamHyper())
    pool.finish_step()
    rows = tl.end()
    ev = [(r, e, s) for _, r, e, s in rows]
    for b in range(2):
        assert ("gpu", "fwd_start", f"block={b}") in ev and ("gpu", "bwd_end", f"block={b}") in ev
    t = {(e, s): ns for ns, _, e, s in rows}
    assert t[("fwd_end", "block=1")] <= t[("bwd_start", "block=1")] <= t[("bwd_end", "block=0")]
    for c in (2, 3):   # pooled chunks (1-based): fetched, drained, updated on the host
        assert sum(1 for r in ev if r == ("h2d", "upload_start", f"chunk={c}")) >= 1
        assert ("d2h", "offload_end", f"chunk={c}") in ev
        assert ("cpu", "update_end", f"chunk={c}") in ev
    assert ("gpu", "optim_end", "chunk=1") in ev
    path = str(tmp_path / "tl.csv")
    write_csv(rows, path)
    assert read_csv(path) == rows
    summ = summarize(rows)
    assert summ["bwd_end_ns"] >= summ["fwd_end_ns"] > 0 and summ["busy_ns"]["cpu"] > 0


@pytest.mark.parametrize("n_persist", [3, 1])
def test_overlapped_chunk_step_is_bit_identical(tmp_path, cuda_device, n_persist):
    """train_step(overlap=True): each persistent chunk's update runs on a side
    stream as soon as its gradients are complete, during the rest of the
    backward. Losses, fp32 masters and bf16 parameters must equal the
    step-after-backward run bit for bit (also with non-persistent chunks,
    whose host Adam must see the same step numbers)."""
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.offload import ChunkPool
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, train_step
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps({"hidden_size": 256, "n_blocks": 2, "n_heads": 4,
                                "vocab_size": 1000, "seq_len": 128}))
    tpath = planner.trace_file(["--spec", str(spec), "--batch", "4"], str(tmp_path / "t.json"))
    trace = json.load(open(tpath))
    layout = planner.pack(tpath, grid="2Mi")
    numels = [c["used_bytes"] // 2 for c in layout["chunks"]]

    def run(overlap):
        cs = ChunkSet(numels[:n_persist], device=cuda_device)
        pool = (ChunkPool(numels, n_persist, 1, device=cuda_device)
                if n_persist < len(numels) else None)
        model = ChunkedGPT2(GPT2Shape.from_trace(trace), layout, cs, trace["ops"], pool=pool)
        model.init_weights(0)
        g = torch.Generator(device=cuda_device).manual_seed(0)
        losses = []
        for _ in range(4):
            x = torch.randint(0, 1000, (4, 128), device=cuda_device, generator=g)
            losses.append(float(train_step(model, x, (x + 1) % 1000,
                                           AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True),
                                           overlap=overlap)))
        torch.cuda.synchronize()
        if pool is not None:
            pool.finish_step()
        state = [t.clone() for c in cs.chunks for t in (c.master, c.exp_avg, c.param)]
        if pool is not None:
            state += [pool.h_master[c].clone() for c in sorted(pool.numel)]
        return losses, state, cs.grad_stats()

    ref_l, ref_s, ref_stats = run(False)
    l, s, stats = run(True)
    assert l == ref_l
    for a, b in zip(s, ref_s):
        assert torch.equal(a.view(torch.int16) if a.dtype == torch.bfloat16 else a,
                           b.view(torch.int16) if b.dtype == torch.bfloat16 else b)
    assert stats[1] == ref_stats[1] and abs(stats[0] - ref_stats[0]) <= 1e-9 * ref_stats[0]


def test_pool_decisions_match_the_simulator(tmp_path, cuda_device):
    """Buffer-pool semantics: the real iteration's chunk
    uploads (h2d stream), drains (d2h stream) and evictions happen in the
    same per-stream order, for the same chunks, as in `memplan simulate` of
    the same plan (one fetch in flight, farthest-next-use eviction, drain
    after the chunk's last backward use)."""
    import subprocess
    from paper_2406_08334_b200 import planner
    from paper_2406_08334_b200.chunks import AdamHyper, ChunkSet
    from paper_2406_08334_b200.offload import ChunkPool
    from paper_2406_08334_b200.timeline import Timeline, read_csv
    from paper_2406_08334_b200.train import ChunkedGPT2, GPT2Shape, train_step
    spec = tmp_path / "spec.json"
    spec.write_text(json.dumps({"hidden_size": 256, "n_blocks": 5, "n_heads": 4,
                                "vocab_size": 1000, "seq_len": 128}))
    tpath = planner.trace_file(["--spec", str(spec), "--batch", "4"], str(tmp_path / "t.json"))
    trace = json.load(open(tpath))
    layout = planner.pack(tpath, grid="2Mi")
    numels = [c["used_bytes"] // 2 for c in layout["chunks"]]
    n_persist, n_buffer = 1, 2
    cs = ChunkSet(numels[:n_persist], device=cuda_device)
    pool = ChunkPool(numels, n_persist, n_buffer, device=cuda_device)
    model = ChunkedGPT2(GPT2Shape.from_trace(trace), layout, cs, trace["ops"], pool=pool)
    model.init_weights(0)
    x = torch.randint(0, 1000, (4, 128), device=cuda_device)
    train_step(model, x, (x + 1) % 1000, AdamHyper())
    pool.finish_step()
    tl = Timeline()
    model.timeline = cs.timeline = pool.timeline = tl
    tl.begin()
    train_step(model, x, (x + 1) % 1000, AdamHyper())
    pool.finish_step()
    real = tl.end()
    memplan = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "build", "memplan")
    sim_csv = str(tmp_path / "sim.csv")
    subprocess.run([memplan, "simulate", "--trace", tpath, "--hw", "a100x1", "--s-chunk",
                    str(layout["s_chunk"]), "--n-persist", str(n_persist), "--n-buffer",
                    str(n_buffer), "--timeline-csv", sim_csv], check=True, capture_output=True)
    sim = read_csv(sim_csv)

    def per_stream(rows, event):
        return [s for _, _, e, s in rows if e == event]

    assert len(numels) - n_persist >= 3   # several pooled chunks, so evictions happen
    for event in ("upload_start", "offload_start", "evict"):
        assert per_stream(real, event) == per_stream(sim, event), event
    assert per_stream(real, "evict")


@pytest.mark.parametrize("checkpoint", [False, True])
def test_graphed_train_step_is_bit_identical(tmp_path, cuda_device, checkpoint):
    """GraphedTrainStep (forward + backward captured in a CUDA graph, chunk
    step eager) trains exactly like train_step: losses, masters and params
    bit for bit, with and without a checkpointed block."""
    from paper_2406_08334_b200.chunks import AdamHyper
    from paper_2406_08334_b200.train import GraphedTrainStep, train_step
    hyper = AdamHyper(lr=1e-3, weight_decay=0.01, adamw=True)

    def run(graphed):
        model, shape = _setup(tmp_path / ("g" if graphed else "e"), cuda_device)
        if checkpoint:
            model.set_block_schedule(["checkpoint", "none"])
        g = torch.Generator(device=cuda_device).manual_seed(0)
        xs = [torch.randint(0, shape.vocab, (4, shape.seq), device=cuda_device, generator=g)
              for _ in range(4)]
        step = GraphedTrainStep(model, xs[0], (xs[0] + 1) % shape.vocab) if graphed else None
        losses = []
        for x in xs:
            y = (x + 1) % shape.vocab
            losses.append(float(step(x, y, hyper) if graphed else train_step(model, x, y, hyper)))
        torch.cuda.synchronize()
        return losses, [t.clone() for c in model.chunks.chunks for t in (c.master, c.param)]

    (tmp_path / "g").mkdir()
    (tmp_path / "e").mkdir()
    ref_l, ref_s = run(False)
    l, s = run(True)
    assert l == ref_l
    for a, b in zip(s, ref_s):
        assert torch.equal(a.view(torch.int16) if a.dtype == torch.bfloat16 else a,
                           b.view(torch.int16) if b.dtype == torch.bfloat16 else b)


def test_model_and_chunks_are_freed(tmp_path, cuda_device):
    """A ChunkedGPT2 and its chunk buffers are released once dropped (no
    reference cycle through the gradient hooks, which live in C++ autograd
    metadata where Python's collector cannot see them)."""
    import gc
    from paper_2406_08334_b200.chunks import AdamHyper
    from paper_2406_08334_b200.train import train_step
    def one_model():
        model, shape = _setup(tmp_path, cuda_device)
        x = torch.randint(0, shape.vocab, (4, shape.seq), device=cuda_device)
        train_step(model, x, (x + 1) % shape.vocab, AdamHyper())
        held = torch.cuda.memory_allocated()
        del model
        gc.collect()
        torch.cuda.synchronize()
        return held

    one_model()   # first use of cuBLAS etc. allocates process-lifetime workspaces
    gc.collect()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    held = one_model()
    assert held > base
    assert torch.cuda.memory_allocated() <= base + (1 << 20)


def test_bias_linear_matches_f_linear(cuda_device):
    """_BiasLinear (bias gradient as a GEMV) gives F.linear's output exactly
    and its gradients within bf16 rounding of the reduction order."""
    from paper_2406_08334_b200.train import _BiasLinear
    g = torch.Generator(device=cuda_device).manual_seed(0)
    x = torch.randn(4, 256, 320, device=cuda_device, dtype=torch.bfloat16, generator=g)
    w = torch.randn(480, 320, device=cuda_device, dtype=torch.bfloat16, generator=g) * 0.05
    b = torch.randn(480, device=cuda_device, dtype=torch.bfloat16, generator=g)
    gy = torch.randn(4, 256, 480, device=cuda_device, dtype=torch.bfloat16, generator=g)
    outs = []
    for fn in (lambda x, w, b: torch.nn.functional.linear(x, w, b), _BiasLinear.apply):
        xx, ww, bb = (t.detach().clone().requires_grad_(True) for t in (x, w, b))
        y = fn(xx, ww, bb)
        y.backward(gy)
        outs.append((y.detach(), xx.grad, ww.grad, bb.grad))
    (y0, gx0, gw0, gb0), (y1, gx1, gw1, gb1) = outs
    assert torch.equal(y0, y1)
    for a, c in ((gx0, gx1), (gw0, gw1), (gb0, gb1)):
        torch.testing.assert_close(a.float(), c.float(), rtol=2e-2, atol=2e-2)
