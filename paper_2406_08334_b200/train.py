"""End-to-end chunked training step: a GPT-2 shaped decoder whose parameters
live in the planner's chunk buffers, trained with the B200 chunk data plane.

The model is exactly the operator sequence the reference synthesizes for the
trace (proj/src/trace.cpp:213-242,316-340): embedding (token + learned
position), per block {attn_norm, attn_qkv, attn_core, attn_out, mlp_norm,
mlp_up, mlp_act, mlp_down}, tied lm_head, cross-entropy. (Like the trace it
has no final LayerNorm.) Parameters are views into the chunk buffers of the
`ChunkLayout` computed by the planner, in execution order — parameter bytes of
op i start at the prefix sum of param_bytes within its chunk (SURVEY §8(a)
a9) — so the chunk the data plane updates is byte-for-byte the chunk the
planner packed.

One iteration (ZeRO-3 chunk semantics):
  1. parameters are the gathered bf16 chunk buffers (all-gathered at the end
     of the previous step);
  2. forward + backward in PyTorch (cuBLAS GEMMs / SDPA attention: the only
     tensor-core work of the step); each parameter's gradient is
     copied into its slot of the chunk's flat bf16 gradient buffer by a
     post-accumulate hook;
  3. the chunk step — reduce-scatter -> fused Adam -> all-gather — through the
     C-ABI (ChunkSet.step).
"""
from __future__ import annotations

import math
import weakref
from dataclasses import dataclass

import torch
import torch.nn.functional as F
import torch.utils.checkpoint

from .chunks import AdamHyper, ChunkSet

BF16 = torch.bfloat16


@dataclass
class GPT2Shape:
    """Decoder shape of a trace. Defaults are GPT-2 (biases, 4h MLP, tied
    embeddings, learned positions); the Llama family of the reference's
    presets (proj/src/presets.cpp:24-37) is gated (SwiGLU), bias-free
    (RMSNorm), untied, rotary, with grouped KV heads."""
    hidden: int = 1600
    blocks: int = 48
    heads: int = 25
    vocab: int = 50257
    seq: int = 1024
    ffn: int = 0          # 0 -> 4 * hidden
    kv_heads: int = 0     # 0 -> heads
    gated: bool = False
    bias: bool = True
    tied: bool = True
    learned_pos: bool = True

    @property
    def ffn_dim(self) -> int:
        return self.ffn or 4 * self.hidden

    @property
    def kv_dim(self) -> int:
        return (self.hidden // self.heads) * (self.kv_heads or self.heads)

    @staticmethod
    def from_trace_meta(meta: dict, n_blocks: int) -> "GPT2Shape":
        return GPT2Shape(int(meta["hidden_size"]), n_blocks, int(meta["n_heads"]),
                         int(meta["vocab_size"]), int(meta["seq_len"]))

    @staticmethod
    def from_trace(trace: dict) -> "GPT2Shape":
        """Recover the architecture from the trace's parameter bytes (the
        meta carries only hidden/heads/vocab/seq, proj/src/trace.cpp:275-282)."""
        meta, ops = trace["meta"], trace["ops"]
        h, heads = int(meta["hidden_size"]), int(meta["n_heads"])
        v, s = int(meta["vocab_size"]), int(meta["seq_len"])
        dt = int(meta.get("dtype_bytes", 2))
        p = {o["name"].split(".")[0]: o["param_bytes"] // dt for o in ops if o["name"].endswith(".0")
             or "." not in o["name"]}
        bias = p["attn_norm"] == 2 * h
        qkv = p["attn_qkv"] // (h + (1 if bias else 0))  # h + 2*kv_dim
        kv_dim = (qkv - h) // 2
        up = p["mlp_up"] // (h + (1 if bias else 0))
        down_f = (p["mlp_down"] - (h if bias else 0)) // h
        gated = up == 2 * down_f
        learned = p["embedding"] == (v + s) * h
        tied = p["lm_head"] == 0
        head_dim = h // heads
        return GPT2Shape(h, trace["n_blocks"], heads, v, s, ffn=down_f,
                         kv_heads=kv_dim // head_dim, gated=gated, bias=bias, tied=tied,
                         learned_pos=learned)


def op_param_shapes(shape: GPT2Shape) -> list[tuple[str, list[tuple[str, tuple[int, ...]]]]]:
    """(op name, [(param name, shape)...]) in trace order, weights then biases
    per op, as synthesize_trace counts them (proj/src/trace.cpp:213-242,316-340)."""
    h, v, s, f, kv = shape.hidden, shape.vocab, shape.seq, shape.ffn_dim, shape.kv_dim
    up = 2 * f if shape.gated else f

    def wb(name, out, inp):
        return [(f"{name}_w", (out, inp))] + ([(f"{name}_b", (out,))] if shape.bias else [])

    def norm(name):
        return [(f"{name}_w", (h,))] + ([(f"{name}_b", (h,))] if shape.bias else [])

    emb = [("wte", (v, h))] + ([("wpe", (s, h))] if shape.learned_pos else [])
    ops = [("embedding", emb)]
    for b in range(shape.blocks):
        ops += [
            (f"attn_norm.{b}", norm("ln1")),
            (f"attn_qkv.{b}", wb("qkv", h + 2 * kv, h)),
            (f"attn_core.{b}", []),
            (f"attn_out.{b}", wb("out", h, h)),
            (f"mlp_norm.{b}", norm("ln2")),
            (f"mlp_up.{b}", wb("up", up, h)),
            (f"mlp_act.{b}", []),
            (f"mlp_down.{b}", wb("down", h, f)),
        ]
    ops += [("lm_head", [] if shape.tied else [("head_w", (v, h))]), ("cross_entropy", [])]
    return ops


class ChunkedGPT2:
    """GPT-2 whose parameters are views into a ChunkSet's gathered buffers."""

    def __init__(self, shape: GPT2Shape, layout: dict, chunks: ChunkSet, trace_ops: list[dict],
                 pool=None):
        """`chunks` holds the persistent chunks (all of them without a pool);
        `pool` (offload.ChunkPool) the non-persistent chunks pool.first.."""
        self.shape = shape
        self.chunks = chunks
        self.pool = pool
        specs = op_param_shapes(shape)
        if len(specs) != len(trace_ops):
            raise ValueError(f"model has {len(specs)} ops, trace has {len(trace_ops)}")
        # op index -> chunk (the layout's spans), then prefix offsets in op order
        chunk_of = {}
        for c in layout["chunks"]:
            for i in range(c["first_op"], c["last_op"] + 1):
                chunk_of[i] = c["chunk_id"]
        offset = [0] * len(layout["chunks"])
        self.params: dict[str, torch.Tensor] = {}
        self.blocks: list[dict[str, torch.Tensor]] = [dict() for _ in range(shape.blocks)]
        self._hooks = []
        # overlapped step (train_step(..., overlap=True)): per persistent
        # chunk, how many parameters must report a gradient before its update
        self._chunk_nparams = [0] * len(chunks.chunks)
        self._pending: list[int] = []
        self._overlap = False
        # non-persistent chunks: parameter specs for ChunkGather, where each
        # param goes (None = top level, else block id), and init staging
        first_pooled = pool.first if pool is not None else len(layout["chunks"])
        self.pool_specs: dict[int, list] = {}
        self.pool_keys: dict[int, list] = {}
        self._init_buf: dict[int, torch.Tensor] = {}
        self.block_chunk = [None] * shape.blocks
        for i, ((name, plist), top) in enumerate(zip(specs, trace_ops)):
            assert top["name"] == name, (top["name"], name)
            n_el = sum(math.prod(s) for _, s in plist)
            assert 2 * n_el == top["param_bytes"], (name, 2 * n_el, top["param_bytes"])
            ci = chunk_of[i]
            where = int(name.split(".")[1]) if "." in name else None
            if where is not None:
                self.block_chunk[where] = ci
            for pname, pshape in plist:
                numel = math.prod(pshape)
                lo = offset[ci]
                offset[ci] += numel
                if ci < first_pooled:
                    cs = chunks.chunks[ci]
                    p = cs.param[lo:lo + numel].view(pshape)
                    p.requires_grad_(True)
                    g = cs.grad[lo:lo + numel].view(pshape)
                    self._hooks.append(p.register_post_accumulate_grad_hook(
                        _stash_into(g, weakref.ref(self), ci)))
                    self._chunk_nparams[ci] += 1
                else:
                    buf = self._init_buf.setdefault(
                        ci, torch.zeros(pool.shard[ci] * pool.world, dtype=BF16,
                                        device=pool.device))
                    p = buf[lo:lo + numel].view(pshape)  # init-time stand-in only
                    self.pool_specs.setdefault(ci, []).append((lo, pshape))
                    self.pool_keys.setdefault(ci, []).append((where, pname))
                if where is not None:
                    self.blocks[where][pname] = p
                else:
                    self.params[pname] = p
        self.wte_chunk = chunk_of[0]
        self.head_chunk = chunk_of[len(specs) - 2]  # the lm_head operator's chunk
        self.anchors = {c: torch.zeros((), device=pool.device, requires_grad=True)
                        for c in self.pool_specs} if pool is not None else {}
        for ci, c in enumerate(layout["chunks"]):
            assert 2 * offset[ci] == c["used_bytes"], "chunk payload mismatch"

    def init_weights(self, seed: int = 0) -> None:
        """GPT-2 / Llama style init, written straight into the chunk buffers;
        the fp32 master copies are refreshed from them."""
        dev = self.chunks.device if self.chunks.chunks or self.pool is None else self.pool.device
        g = torch.Generator(device=dev).manual_seed(seed)
        std = 0.02
        with torch.no_grad():
            for name in ("wte", "wpe", "head_w"):
                if name in self.params:
                    self.params[name].normal_(0.0, std, generator=g)
            for blk in self.blocks:
                for k, p in blk.items():
                    if k.endswith("_w") and p.dim() == 2:
                        s = std / math.sqrt(2 * self.shape.blocks) if k in ("out_w", "down_w") else std
                        p.normal_(0.0, s, generator=g)
                    elif k in ("ln1_w", "ln2_w"):
                        p.fill_(1.0)
                    else:
                        p.zero_()
            for c in self.chunks.chunks:
                c.master.copy_(c.param_shard().float())
                c.exp_avg.zero_()
                c.exp_avg_sq.zero_()
            for ci, buf in self._init_buf.items():  # non-persistent: to the host shards
                self.pool.load_initial(ci, buf)
                for where, pname in self.pool_keys[ci]:  # drop the init stand-ins
                    (self.params if where is None else self.blocks[where])[pname] = None
        self._init_buf.clear()

    timeline = None   # timeline.Timeline: per-block fwd/bwd events (simulator schema)

    def _block_start(self, b: int, x: torch.Tensor) -> None:
        tl = getattr(self, "timeline", None)
        if tl is None:
            return
        tl.gpu(None, "gpu", "fwd_start", f"block={b}")
        if x.requires_grad:  # grad of the block input ready = the block's backward done
            x.register_hook(lambda g, b=b: tl.gpu(None, "gpu", "bwd_end", f"block={b}"))

    def _block_end(self, b: int, x: torch.Tensor) -> None:
        tl = getattr(self, "timeline", None)
        if tl is None:
            return
        tl.gpu(None, "gpu", "fwd_end", f"block={b}")
        if x.requires_grad:  # grad of the block output ready = its backward starts
            x.register_hook(lambda g, b=b: tl.gpu(None, "gpu", "bwd_start", f"block={b}"))

    def _strategies(self) -> list[str]:
        return getattr(self, "strategies", None) or ["none"] * self.shape.blocks

    def pool_uses(self) -> dict[int, int]:
        """ChunkGather nodes per non-persistent chunk in one forward: one
        shared by the chunk's plain operators, one per checkpointed block (its
        gather lives inside the recomputable function), and one more for the
        tied embedding's chunk at the head."""
        strategies = self._strategies()
        uses = {c: 0 for c in self.pool_specs}
        plain = {self.wte_chunk} | {self.block_chunk[b] for b, st in enumerate(strategies)
                                    if st != "checkpoint"}
        if not self.shape.tied:
            plain.add(self.head_chunk)
        for c in uses:
            uses[c] += 1 if c in plain else 0
        for b, st in enumerate(strategies):
            if st == "checkpoint" and self.block_chunk[b] in uses:
                uses[self.block_chunk[b]] += 1
        if self.shape.tied and self.wte_chunk in uses:
            uses[self.wte_chunk] += 1
        return {c: n for c, n in uses.items() if n > 0}

    def _loss_pooled(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        from .offload import ChunkGather
        sh, pool = self.shape, self.pool
        params = dict(self.params)
        blocks = [dict(b) for b in self.blocks]
        done: set[int] = set()

        def gather_into(c, position, prefetch, p_dict, b_list):
            outs = ChunkGather.apply(self.anchors[c], pool, c, self.pool_specs[c], position,
                                     prefetch)
            for (where, pname), t in zip(self.pool_keys[c], outs):
                (p_dict if where is None else b_list[where])[pname] = t

        def ensure(c):  # forward reaches chunk c: gather it, prefetch c+1
            if c in self.pool_specs and c not in done:
                gather_into(c, c + 1, c + 1, params, blocks)
                done.add(c)

        def checkpointed(blk_id):
            c = self.block_chunk[blk_id]

            def fn(x):
                # the gather is part of the recomputed function: the recompute
                # in backward re-acquires the chunk (it may have been evicted)
                local = [dict(b) for b in blocks]
                if c in self.pool_specs:
                    gather_into(c, c + 1, c + 1, {}, local)
                return block_forward(sh, local[blk_id], x)
            return fn

        ensure(self.wte_chunk)
        x = embed(sh, params, tokens)
        strategies = self._strategies()
        swap_blocks = [b for b, st in enumerate(strategies) if st == "swap"]
        for blk_id, strategy in enumerate(strategies):
            if strategy == "checkpoint":
                self._block_start(blk_id, x)
                x = torch.utils.checkpoint.checkpoint(checkpointed(blk_id), x, use_reentrant=False)
            else:
                ensure(self.block_chunk[blk_id])
                self._block_start(blk_id, x)
                if strategy == "swap":
                    self._swap.begin_block(blk_id)
                    with torch.autograd.graph.saved_tensors_hooks(self._swap.pack,
                                                                  self._swap.unpack):
                        x = block_forward(sh, blocks[blk_id], x)
                else:
                    x = block_forward(sh, blocks[blk_id], x)
            self._block_end(blk_id, x)
            if swap_blocks:
                self._swap.prefetch_hooks(swap_blocks, blk_id, x, blk_id == len(strategies) - 1)
        if sh.tied and self.wte_chunk in self.pool_specs:  # tied head: another use of chunk 0
            gather_into(self.wte_chunk, pool.n_total, None, params, blocks)
        elif not sh.tied:
            ensure(self.head_chunk)
        return head_loss(sh, params, x, targets)

    def set_block_schedule(self, strategies: list[str]) -> None:
        """Per-block activation policy from the planner's BlockSchedule
        ("swap" | "checkpoint" | "none", proj/src/layout.cpp:218-249):
        checkpoint = recompute the block in backward; swap = its saved
        activations go to pinned host memory on a side stream after use in
        forward and come back before its backward (parameters stay put)."""
        if len(strategies) != self.shape.blocks:
            raise ValueError("one strategy per block")
        self.strategies = list(strategies)
        self._swap = ActivationSwap({c.param.untyped_storage().data_ptr()
                                     for c in self.chunks.chunks}, getattr(self, "pool", None))
        self._swap.set_lead([b for b, st in enumerate(self.strategies) if st == "swap"])

    def loss(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        pool = getattr(self, "pool", None)
        if pool is not None:
            with torch.autograd.graph.saved_tensors_hooks(pool.pack, pool.unpack):
                return self._loss_pooled(tokens, targets)
        sh = self.shape
        x = embed(sh, self.params, tokens)
        strategies = getattr(self, "strategies", None) or ["none"] * len(self.blocks)
        swap_blocks = [b for b, st in enumerate(strategies) if st == "swap"]
        for b, (blk, strategy) in enumerate(zip(self.blocks, strategies)):
            ChunkedGPT2._block_start(self, b, x)   # (tests call loss on a plain namespace)
            if strategy == "checkpoint":
                x = torch.utils.checkpoint.checkpoint(block_forward, sh, blk, x, use_reentrant=False)
            elif strategy == "swap":
                self._swap.begin_block(b)
                with torch.autograd.graph.saved_tensors_hooks(self._swap.pack, self._swap.unpack):
                    x = block_forward(sh, blk, x)
            else:
                x = block_forward(sh, blk, x)
            ChunkedGPT2._block_end(self, b, x)
            if swap_blocks:
                self._swap.prefetch_hooks(swap_blocks, b, x, b == len(strategies) - 1)
        return head_loss(sh, self.params, x, targets)


def embed(sh: GPT2Shape, params: dict, tokens: torch.Tensor) -> torch.Tensor:
    """The trace's `embedding` operator (token + learned position, or token
    only for rotary models)."""
    x = F.embedding(tokens, params["wte"])
    if sh.learned_pos:
        x = x + params["wpe"][: tokens.shape[1]]
    return x


def head_logits(sh: GPT2Shape, params: dict, x: torch.Tensor) -> torch.Tensor:
    """`lm_head` (tied to the embedding, or its own weight), after a final
    norm WITHOUT affine parameters: the reference's traces carry no final-norm
    operator (proj/src/trace.cpp:320-340 -- embedding, 8 ops per block,
    lm_head, cross_entropy), so the parameter bytes stay the trace's, while
    the residual stream is still normalised before the vocabulary projection
    (without it the 48-block stream makes the first Adam steps unstable).

    GPT-2's vocabulary (50257) is not a multiple of 8, and with that
    leading dimension cuBLAS falls back to `align1` SM75 mma.sync GEMMs for
    the projection and both its gradients (28 of 136 ms of a GPT-2 1.5B
    iteration, scripts/train_breakdown.py). The weight is therefore padded
    with zero rows to a multiple of 64 for the GEMM (a 160 MB copy) and the
    logits sliced back: the same values, aligned kernels."""
    x = _norm(sh, x, None, None)
    w = params["wte"] if sh.tied else params["head_w"]
    pad = (-w.shape[0]) % 64
    if pad == 0:
        return F.linear(x, w)
    return F.linear(x, F.pad(w, (0, 0, 0, pad)))[..., : w.shape[0]]


def head_loss(sh: GPT2Shape, params: dict, x: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
    logits = head_logits(sh, params, x)
    return F.cross_entropy(logits.view(-1, sh.vocab).float(), targets.reshape(-1))


_ROPE_CACHE: dict = {}


def _rope(x: torch.Tensor) -> torch.Tensor:
    """Rotary position embedding on (b, s, heads, head_dim), half-split form."""
    s, d = x.shape[1], x.shape[-1]
    key = (s, d, x.device, x.dtype)
    if key not in _ROPE_CACHE:
        inv = 1.0 / (10000 ** (torch.arange(0, d, 2, device=x.device, dtype=torch.float32) / d))
        ang = torch.outer(torch.arange(s, device=x.device, dtype=torch.float32), inv)
        _ROPE_CACHE[key] = (ang.cos()[None, :, None, :].to(x.dtype),
                            ang.sin()[None, :, None, :].to(x.dtype))
    cos, sin = _ROPE_CACHE[key]
    x1, x2 = x[..., : d // 2], x[..., d // 2:]
    return torch.cat((x1 * cos - x2 * sin, x2 * cos + x1 * sin), dim=-1)


def _norm(sh: GPT2Shape, x, w, b):
    if sh.bias:
        return F.layer_norm(x, (sh.hidden,), w, b)
    return F.rms_norm(x, (sh.hidden,), w)


class _BiasLinear(torch.autograd.Function):
    """y = x W^T + b with the bias gradient as a GEMV (ones^T dY on cuBLAS)
    instead of a column-sum reduction kernel over the (tokens x out) output
    gradient: the reductions took 5.9 ms of a GPT-2 1.5B iteration
    (scripts/train_breakdown.py). Forward and the x / W gradients are the
    same GEMMs F.linear runs."""

    @staticmethod
    def forward(ctx, x, w, b):
        ctx.save_for_backward(x, w)
        return F.linear(x, w, b)

    @staticmethod
    def backward(ctx, gy):
        x, w = ctx.saved_tensors
        gy2 = gy.reshape(-1, gy.shape[-1])
        gx = gw = gb = None
        if ctx.needs_input_grad[0]:
            gx = (gy2 @ w).view(x.shape)
        if ctx.needs_input_grad[1]:
            gw = gy2.t() @ x.reshape(-1, x.shape[-1])
        if ctx.needs_input_grad[2]:
            ones = torch.ones(1, gy2.shape[0], dtype=gy2.dtype, device=gy2.device)
            gb = (ones @ gy2).view(-1)
        return gx, gw, gb


def _linear(x, w, b):
    return F.linear(x, w) if b is None else _BiasLinear.apply(x, w, b)


def block_forward(sh: GPT2Shape, blk: dict, x: torch.Tensor, mark=None) -> torch.Tensor:
    """One transformer block: the trace's attn_norm .. mlp_down operators.
    GPT-2: LayerNorm, fused QKV with bias, GELU MLP. Llama: RMSNorm, rotary
    q/k, grouped KV heads, SwiGLU MLP, no biases.
    `mark(k, out)` (profiler only) is called after operator k with its output."""
    mark = mark or (lambda k, out: out)
    b, s, _ = x.shape
    hd = sh.hidden // sh.heads
    kvh = sh.kv_heads or sh.heads
    y = mark(0, _norm(sh, x, blk["ln1_w"], blk.get("ln1_b")))
    qkv = mark(1, _linear(y, blk["qkv_w"], blk.get("qkv_b")))
    q, k, v = qkv.split([sh.hidden, sh.kv_dim, sh.kv_dim], dim=-1)
    q, k, v = q.view(b, s, sh.heads, hd), k.view(b, s, kvh, hd), v.view(b, s, kvh, hd)
    if not sh.learned_pos:
        q, k = _rope(q), _rope(k)
    a = mark(2, F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2),
                                               v.transpose(1, 2), is_causal=True,
                                               enable_gqa=kvh != sh.heads))
    x = mark(3, x + _linear(a.transpose(1, 2).reshape(b, s, sh.hidden), blk["out_w"],
                             blk.get("out_b")))
    y = mark(4, _norm(sh, x, blk["ln2_w"], blk.get("ln2_b")))
    y = mark(5, _linear(y, blk["up_w"], blk.get("up_b")))
    if sh.gated:
        gate, up = y.chunk(2, dim=-1)
        y = mark(6, F.silu(gate) * up)
    else:
        y = mark(6, F.gelu(y, approximate="tanh"))
    return mark(7, x + _linear(y, blk["down_w"], blk.get("down_b")))


class ActivationSwap:
    """saved_tensors_hooks for Swap blocks: each saved activation is copied to
    pinned host memory on a side stream (swap-out overlapping the forward),
    its device memory released to the allocator once that copy is done
    (record_stream). In backward the block's activations come back ahead of
    need: `prefetch(b)` -- fired by a gradient hook when backward reaches
    block b + `lead` -- issues all of block b's H2D copies on the side stream,
    so by the time autograd unpacks them the compute stream only waits on
    their events (the simulator's swap-in before the block's backward,
    proj/src/sim.cpp:411-425). A tensor unpacked before its prefetch is copied
    on demand. Tensors that live in the chunk buffers (parameters) are never
    swapped; parameters of non-persistent chunks (pool slots) are handed to
    the pool's own hooks."""

    lead = 2   # prefetch block b when the backward of block b + lead starts (see set_lead)

    def __init__(self, param_storages: set[int], pool=None):
        self.params = param_storages
        self.pool = pool
        self.side = torch.cuda.Stream()
        self.block = None
        self.saved: dict[int, list[dict]] = {}
        self.timeline = None

    def set_lead(self, swap_blocks: list[int]) -> None:
        """Prefetch distance in blocks (default 2; PTK_SWAP_LEAD overrides).
        Measured both ways: a longer lead helped a GPT-2 10B plan (lead 4:
        -3..5 %) and hurt a Llama-2 13B plan sized to the last GB (lead 3:
        +14 %, the prefetched block competes for memory and host DRAM), so
        the default stays 2 (profiles/README.md)."""
        import os
        self.lead = max(1, int(os.environ.get("PTK_SWAP_LEAD", "2")))

    def begin_block(self, b: int) -> None:
        self.block = b
        self.saved[b] = []

    def pack(self, t: torch.Tensor):
        if self.pool is not None and t.untyped_storage().data_ptr() in self.pool._slot_ptr:
            return ("pool", self.pool.pack(t))
        if not t.is_cuda or t.untyped_storage().data_ptr() in self.params:
            return ("keep", t)
        cur = torch.cuda.current_stream()
        self.side.wait_stream(cur)
        with torch.cuda.stream(self.side):
            host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            host.copy_(t, non_blocking=True)
        t.record_stream(self.side)
        entry = {"host": host, "device": t.device, "dev": None, "ev": None}
        self.saved.setdefault(self.block, []).append(entry)
        return ("swap", entry)

    def _fetch(self, entry: dict) -> None:
        with torch.cuda.stream(self.side):
            entry["dev"] = entry["host"].to(entry["device"], non_blocking=True)
            entry["ev"] = torch.cuda.Event()
            entry["ev"].record(self.side)

    def prefetch(self, b: int) -> None:
        entries = self.saved.pop(b, [])
        if not entries:
            return
        self.side.wait_stream(torch.cuda.current_stream())
        tl = self.timeline
        if tl is not None:
            tl.gpu(self.side, "h2d", "swap_in_start", f"block={b}")
        for entry in entries:
            if entry["dev"] is None:
                self._fetch(entry)
        if tl is not None:
            tl.gpu(self.side, "h2d", "swap_in_end", f"block={b}")

    def unpack(self, packed):
        if packed[0] == "keep":
            return packed[1]
        if packed[0] == "pool":
            return self.pool.unpack(packed[1])
        entry = packed[1]
        cur = torch.cuda.current_stream()
        if entry["dev"] is None:   # not prefetched: copy now
            self.side.wait_stream(cur)
            self._fetch(entry)
        cur.wait_event(entry["ev"])
        dev = entry["dev"]
        dev.record_stream(cur)
        return dev

    def prefetch_hooks(self, swap_blocks: list[int], j: int, x: torch.Tensor,
                       last: bool) -> None:
        """Called with the output x of block j: its gradient hook prefetches
        every swap block b with b + lead == j (or b + lead beyond the last
        block, on the last block's output)."""
        if not x.requires_grad:
            return
        due = [b for b in swap_blocks if b + self.lead == j or (last and b + self.lead > j)]
        if due:
            x.register_hook(lambda g, due=tuple(due): [self.prefetch(b) for b in due] and None)


def _stash_into(slot: torch.Tensor, model_ref=None, ci: int = -1):
    # The model is held WEAKLY: the hook lives in the parameter's C++ autograd
    # metadata, invisible to Python's cycle collector, so a strong reference
    # back to the model would keep the model -- and its chunk buffers -- alive
    # forever (measured: a 26 GB profiling model never freed).
    def hook(p: torch.Tensor) -> None:
        slot.copy_(p.grad)
        p.grad = None
        model = model_ref() if model_ref is not None else None
        if model is not None and model._overlap:
            model._pending[ci] -= 1
            if model._pending[ci] == 0:   # chunk ci's gradients are complete
                model.chunks.step_chunk_overlapped(ci)
    return hook


def train_step(model: ChunkedGPT2, tokens: torch.Tensor, targets: torch.Tensor,
               hyper: AdamHyper, overlap: bool = False) -> torch.Tensor:
    """One iteration; returns the (device) loss. Gradient slots of the chunk
    buffers are fully overwritten by the hooks each step (padding stays 0).

    overlap=True: each persistent chunk's step (RS -> Adam -> AG) is issued
    on a side stream the moment its last gradient lands, while the backward
    of the earlier blocks continues (a chunk's parameters are used only by
    its own operators, all of which have run backward by then); the results
    are bit-identical to the step after the whole backward."""
    step_no = model.chunks.step_count + 1   # of this iteration, for every chunk
    if overlap:
        if not hasattr(model, "_side"):
            model._side = torch.cuda.Stream(model.chunks.device)
        model._pending = list(model._chunk_nparams)
        model._overlap = True
        model.chunks.begin_overlapped_step(hyper, model._side)
    try:
        return _train_step(model, tokens, targets, hyper, overlap, step_no)
    finally:
        model._overlap = False


def _train_step(model, tokens, targets, hyper, overlap, step_no):
    pool = getattr(model, "pool", None)
    tl = model.timeline
    if pool is not None:
        pool.begin_step(step_no, hyper, model.pool_uses())
    if tl is not None:
        tl.host("host", "forward_call_start", "")
    loss = model.loss(tokens, targets)
    if tl is not None:
        tl.host("host", "forward_call_end", "")
        tl.gpu(None, "gpu", "loss_ready", "")
    loss.backward()
    if tl is not None:
        tl.host("host", "backward_call_end", "")
    if overlap:
        model.chunks.finish_overlapped_step()
    else:
        model.chunks.step(hyper)  # persistent chunks; pooled chunks drained during backward
    return loss.detach()


class GraphedTrainStep:
    """The forward + backward of an all-persistent ChunkedGPT2 captured once
    into a CUDA graph and replayed every iteration (the model's ~40 kernels
    per block no longer pay host launch latency); the chunk step (RS -> Adam
    -> AG through the C-ABI) runs after it, eagerly, with the step's own
    Adam scalars. Parameters and gradient slots are the chunk buffers, so
    the graph's addresses stay valid; tokens / targets are copied into static
    inputs. Bit-identical to train_step (same kernels, same order).

    Requires: no non-persistent chunks (the pool's fetches and host Adam are
    host-synchronising) and no swap blocks (pinned-memory saved-tensor
    hooks); checkpoint blocks are captured as recompute."""

    def __init__(self, model: ChunkedGPT2, tokens: torch.Tensor, targets: torch.Tensor,
                 warmup: int = 2):
        if getattr(model, "pool", None) is not None:
            raise ValueError("graphed step needs every chunk persistent")
        if "swap" in model._strategies():
            raise ValueError("graphed step does not capture activation swap")
        self.model = model
        self.x = tokens.clone()
        self.y = targets.clone()
        side = torch.cuda.Stream(model.chunks.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):   # warm-up outside capture (allocator, cuBLAS handles)
            for _ in range(warmup):
                model.loss(self.x, self.y).backward()
        torch.cuda.current_stream().wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.loss = model.loss(self.x, self.y)
            self.loss.backward()

    def __call__(self, tokens: torch.Tensor, targets: torch.Tensor, hyper: AdamHyper) -> torch.Tensor:
        self.x.copy_(tokens, non_blocking=True)
        self.y.copy_(targets, non_blocking=True)
        self.graph.replay()
        self.model.chunks.step(hyper)
        return self.loss.detach().clone()
