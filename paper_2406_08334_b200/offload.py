"""Non-persistent chunks inside the training model: host-resident shards, a
pool of device buffers, fetch-before-use and drain-after-backward, driven by
autograd instead of a trace. Every residency decision (which slot, which
chunk to evict, when a slot frees up) is made by the runtime's ONE policy
implementation, memplan::ChunkBufferPool in libptk.so (ptk_pool_*; the same
code the simulator and the device executor run, proj/src/sim.cpp:275-451's
rules); this module moves the bytes.

* storage: chunk c >= n_persist keeps its rank shard in pinned host memory
  (fp32 master/m/v, bf16 params, bf16 grads); `n_buffer` device slots hold
  gathered bf16 chunks (the reference's buffer = the working copy only);
* fetch (`acquire`): wait for the chunk's previous host update, H2D of the
  shard into its slot position on the h2d stream (+ NCCL all-gather, w > 1),
  the compute stream waits on that event; one prefetch ahead (the next chunk
  in forward, the previous one in backward);
* eviction (policy): the resident pool chunk whose next use (forward
  position c, backward position 2N-c+1) is farthest, never the chunk being
  acquired or in use; a prefetch is issued only if that chunk is needed
  strictly later than the prefetched one (the simulator's rule). The h2d
  stream waits for all compute issued so far before it overwrites the slot;
* autograd: a chunk's parameters are outputs of `ChunkGather` (one node per
  use in forward); tensors autograd saves that live in a slot are saved as
  (chunk, offset, shape) and re-acquired on unpack, so a chunk evicted between
  its forward and backward is fetched again (re-gather in backward);
* drain: when the gradients of all uses of chunk c have arrived
  (ChunkGather.backward), they are summed in a padded staging tensor,
  reduce-scattered (w > 1), the shard goes D2H on the d2h stream and a worker
  thread runs the host Adam (ptk_cpu_adam — bit-identical to the device rule)
  producing the bf16 shard the next fetch uploads;
* pieces: the shard moves in `piece`-element pieces so the three stages
  overlap inside a chunk — the host Adam of piece k starts as soon as its
  D2H lands, and a fetch that finds the chunk's update still running uploads
  each piece the moment the host has finished it (the chunk is still made
  resident as a whole, as the reference's simulator models it,
  proj/src/sim.cpp:335-368,438-451). The update is elementwise, so piecewise
  results are bit-identical to one call over the shard.
"""
from __future__ import annotations

import ctypes
import os
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import torch

from . import _native as nat
from .chunks import AdamHyper, map_peer_buffers, vp

BF16 = torch.bfloat16


def _sh(stream: torch.cuda.Stream) -> ctypes.c_void_p:
    return ctypes.c_void_p(stream.cuda_stream)


class ChunkPool:
    """`exchange` (w > 1): "nccl" -- NCCL all-gather on fetch and in-place
    bf16 reduce-scatter on drain (needs `comm`); "peer" -- the same two steps
    over NVLink peer memory without a library collective (attach_ipc_peers):
    the fetch pulls every peer's shard out of the peer's slot with
    copy-engine transfers (ptk_peer_allgather), the drain sums the owned
    shard of every rank's gradient in fp32 in rank order
    (ptk_peer_reduce_scatter_f32) and the host Adam consumes that fp32 sum
    (ptk_cpu_adam_f32grad) -- exactly the numbers the fused persistent step
    computes, so an offloaded chunk trains bit-identically to a persistent
    one at any w. Both bracket their transfers with peer barriers (one
    signal array for the h2d stream's gathers, one for the compute stream's
    reduces)."""

    def __init__(self, numels: list[int], first: int, n_buffer: int, world: int = 1, rank: int = 0,
                 comm=None, device=None, cpu_threads: int | None = None,
                 piece: int = 32 * 1024 * 1024, exchange: str = "nccl"):
        if n_buffer < 1:
            raise ValueError("non-persistent chunks need at least one buffer")
        if exchange not in ("nccl", "peer"):
            raise ValueError(f"unknown exchange {exchange!r}")
        if world > 1 and exchange == "nccl" and comm is None:
            raise ValueError("world > 1 needs a ptk_comm communicator")
        self.exchange = exchange
        # the host Adam must not starve the threads that launch the GPU work
        # (Python main thread + autograd's device thread): leave two cores per
        # rank, and split the host between the ranks of this node
        local_world = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))
        self.cpu_threads = cpu_threads or max(1, (os.cpu_count() or 4) // local_world - 2)
        self.device = torch.device(device or "cuda")
        self.first, self.world, self.rank, self.comm = first, world, rank, comm
        self.n_total = len(numels)
        self.numel = {c: numels[c] for c in range(first, len(numels))}
        self.shard = {c: nat.shard_elems(n, world) for c, n in self.numel.items()}
        n_pad_max = max(self.shard[c] * world for c in self.numel)
        pin = dict(device="cpu", pin_memory=True)
        self.h_param = {c: torch.zeros(s, dtype=BF16, **pin) for c, s in self.shard.items()}
        # the offloaded gradient: bf16 (NCCL's in-place reduce-scatter), or the
        # fp32 rank-order sum of the peer exchange
        gdt = torch.float32 if exchange == "peer" else BF16
        self.h_grad = {c: torch.zeros(s, dtype=gdt, **pin) for c, s in self.shard.items()}
        self.h_master = {c: torch.zeros(s, dtype=torch.float32, **pin) for c, s in self.shard.items()}
        self.h_m = {c: torch.zeros(s, dtype=torch.float32, **pin) for c, s in self.shard.items()}
        self.h_v = {c: torch.zeros(s, dtype=torch.float32, **pin) for c, s in self.shard.items()}
        self.slots = [torch.zeros(n_pad_max, dtype=BF16, device=self.device)
                      for _ in range(n_buffer)]
        self.device_bytes = 2 * n_pad_max * n_buffer
        self.host_bytes = sum(16 * s for s in self.shard.values())
        # chunks 0..first-1 are persistent (resident, never pooled)
        self.policy = nat.BufferPool(len(numels), first, n_buffer)
        self.slot_released: list = [None] * n_buffer  # compute event at the slot's release
        self.ready: dict[int, torch.cuda.Event] = {}
        self.h2d, self.d2h = torch.cuda.Stream(self.device), torch.cuda.Stream(self.device)
        self.worker = ThreadPoolExecutor(max_workers=1)
        self.updates: dict[int, object] = {}   # chunk -> Future of its host Adam
        self.piece = max(8, piece // 8 * 8)
        self.piece_done: dict[int, list[threading.Event]] = {}  # chunk -> per-piece host Adam done
        self.position = 0
        self.pending_uses: dict[int, int] = {}
        self.partial: dict[int, torch.Tensor] = {}
        self.hyper = AdamHyper()
        self.step = 0
        self.counters = {"fetch": 0, "evict": 0, "h2d_bytes": 0, "d2h_bytes": 0}
        self.timeline = None   # timeline.Timeline: events in the simulator's schema
        self._lock = threading.RLock()
        self._slot_ptr = {t.untyped_storage().data_ptr(): k for k, t in enumerate(self.slots)}
        if exchange == "peer":
            shard_max = max(self.shard.values())
            # the drained chunk's local gradient, read by every peer's reduce
            self.staging = torch.zeros(n_pad_max, dtype=BF16, device=self.device)
            # this rank's reduced fp32 shard, two buffers so a D2H can still
            # be reading one while the next drain reduces into the other
            self.reduced = [torch.zeros(shard_max, dtype=torch.float32, device=self.device)
                            for _ in range(2)]
            self.reduced_free: list = [None, None]   # d2h event: the buffer's last D2H done
            self.n_drains = 0
            self.slot_peers = self.staging_peers = None
            self.sig_gather = self.sig_reduce = None
            self.g_epoch = self.r_epoch = 0
            if world == 1:   # nothing to exchange: the local buffers are the peer table
                self._set_peer_tables([[t.data_ptr() for t in self.slots] + [self.staging.data_ptr()]])

    # ------------------------------------------------ peer exchange setup --
    def _set_peer_tables(self, ptrs) -> None:
        """ptrs[r] = rank r's [slot 0 .. slot n_buffer-1, staging, (signals...)]
        as mapped in this process."""
        arr = ctypes.c_void_p * nat.PTK_MAX_PEERS
        nb = len(self.slots)
        self.slot_peers = [arr(*[ptrs[r][k] for r in range(self.world)]) for k in range(nb)]
        self.staging_peers = arr(*[ptrs[r][nb] for r in range(self.world)])
        if len(ptrs[0]) > nb + 1:
            self.sig_gather = arr(*[ptrs[r][nb + 1] for r in range(self.world)])
            self.sig_reduce = arr(*[ptrs[r][nb + 2] for r in range(self.world)])

    def attach_ipc_peers(self, group=None) -> None:
        """exchange="peer", w > 1: map every peer's slots, gradient staging
        buffer and the two signal arrays into this process (cudaIpc handles
        exchanged through torch.distributed -- plumbing only). Collective."""
        import torch.distributed as dist
        if self.exchange != "peer":
            raise ValueError("attach_ipc_peers needs exchange='peer'")
        if self.world == 1:
            return
        self._signals = [torch.zeros(nat.PTK_MAX_PEERS, dtype=torch.int32, device=self.device)
                         for _ in range(2)]
        bufs = list(self.slots) + [self.staging] + self._signals
        ptrs, self._opened, _ = map_peer_buffers(bufs, self.world, self.rank, self.device, group)
        self._set_peer_tables(ptrs)
        dist.barrier(group=group)

    def close_ipc_peers(self) -> None:
        for base in getattr(self, "_opened", []):
            nat.lib.ptk_ipc_close_handle(base)
        self._opened = []

    def _barrier(self, sig, stream) -> None:
        if sig is self.sig_gather:
            self.g_epoch += 1
            epoch = self.g_epoch
        else:
            self.r_epoch += 1
            epoch = self.r_epoch
        nat.lib.ptk_peer_barrier(sig, self.world, self.rank, epoch, _sh(stream))

    # ------------------------------------------------------------ storage --
    def load_initial(self, c: int, full_chunk: torch.Tensor) -> None:
        """Initial bf16 parameters of chunk c (the gathered chunk, on device)."""
        s, lo = self.shard[c], self.rank * self.shard[c]
        part = torch.zeros(s, dtype=BF16, device=self.device)
        n = max(0, min(s, full_chunk.numel() - lo))
        part[:n] = full_chunk[lo:lo + n]
        self.h_param[c].copy_(part.cpu())
        self.h_master[c].copy_(part.float().cpu())
        self.h_m[c].zero_()
        self.h_v[c].zero_()

    # -------------------------------------------------------------- policy --
    def resident(self, c: int) -> bool:
        return self.policy.slot_of(c) >= 0

    def _pieces(self, c: int):
        s = self.shard[c]
        return [(lo, min(self.piece, s - lo)) for lo in range(0, s, self.piece)]

    def _fetch(self, c: int, keep: int, blocking: bool = True) -> bool:
        """Issue the fetch of chunk c (host update -> H2D shard -> all-gather).
        A prefetch (blocking=False) never stalls the launching thread on the
        chunk's pending host update: it is skipped and retried later. A
        blocking fetch of a chunk whose update is still running uploads it
        piece by piece as the host finishes each piece."""
        if self.resident(c):
            return True
        fut = self.updates.get(c)
        if fut is not None and not blocking and not fut.done():
            self.counters["prefetch_deferred"] = self.counters.get("prefetch_deferred", 0) + 1
            return False
        # acquiring c itself is a demand fetch (it is needed now); a prefetch
        # follows the simulator's rule (evict only a chunk needed later than c)
        granted = self.policy.grant(c, self.position, pinned=(c, keep), demand=c == keep)
        if granted is None:
            if c == keep:
                raise RuntimeError("chunk pool exhausted: every buffer is in use")
            self.counters["prefetch_refused"] = self.counters.get("prefetch_refused", 0) + 1
            return False
        k, v = granted
        if v is None:
            # compute that used the slot before it was freed must be done
            if self.slot_released[k] is not None:
                self.h2d.wait_event(self.slot_released[k])
        else:
            self.ready.pop(v, None)
            self.counters["evict"] += 1
            if self.timeline is not None:
                self.timeline.gpu(torch.cuda.current_stream(self.device), "gpu", "evict",
                                  f"chunk={v + 1}")
            # the evicted chunk may still be read by compute already issued
            self.h2d.wait_stream(torch.cuda.current_stream(self.device))
        s = self.shard[c]
        dst = self.slots[k][self.rank * s:(self.rank + 1) * s]
        done = self.piece_done.get(c) if fut is not None else None
        waited = 0.0
        if self.timeline is not None:
            self.timeline.gpu(self.h2d, "h2d", "upload_start", f"chunk={c + 1}")
        for i, (lo, n) in enumerate(self._pieces(c)):
            if done is not None and not done[i].is_set():
                t0 = time.perf_counter()
                done[i].wait()   # the previous step's host Adam of this piece
                waited += time.perf_counter() - t0
            nat.lib.ptk_memcpy_h2d_async(vp(dst[lo:]), vp(self.h_param[c][lo:]), 2 * n,
                                         _sh(self.h2d))
        if fut is not None:
            fut.result()   # surfaces a host-side failure
            self.updates.pop(c, None)
            self.counters["host_wait_s"] = self.counters.get("host_wait_s", 0.0) + waited
        self.counters["h2d_bytes"] += 2 * s
        if self.exchange == "peer" and self.world > 1:
            if self.sig_gather is None:
                raise RuntimeError("exchange='peer' needs attach_ipc_peers() before use")
            # every rank's own shard is in its slot k -> pull the others' ->
            # nobody reuses slot k before every peer has finished pulling
            self._barrier(self.sig_gather, self.h2d)
            nat.lib.ptk_peer_allgather(self.slot_peers[k], self.world, self.rank, 2 * s,
                                       _sh(self.h2d))
            self._barrier(self.sig_gather, self.h2d)
        elif self.comm is not None:
            nat.lib.ptk_chunk_allgather(self.comm, vp(self.slots[k]), s, 0, _sh(self.h2d))
        if self.timeline is not None:
            self.timeline.gpu(self.h2d, "h2d", "upload_end", f"chunk={c + 1}")
        ev = torch.cuda.Event()
        ev.record(self.h2d)
        self.ready[c] = ev
        self.policy.arrived(c)  # stream-ordered: users wait on ready[c]
        self.counters["fetch"] += 1
        return True

    def acquire(self, c: int, position: int, prefetch: int | None = None) -> torch.Tensor:
        """Make chunk c resident for the compute stream; returns its gathered
        bf16 buffer (n_pad elements) and starts the prefetch of `prefetch`."""
        with self._lock:
            self.position = position
            self._fetch(c, c)
            torch.cuda.current_stream(self.device).wait_event(self.ready[c])
            view = self.slots[self.policy.slot_of(c)][: self.shard[c] * self.world]
            if prefetch is not None and prefetch in self.numel and not self.resident(prefetch):
                # w > 1: the prefetch's all-gather must be issued in the same
                # order on every rank, so it may not depend on host timing (the
                # policy's decision depends on positions only)
                self._fetch(prefetch, c, blocking=self.world > 1)
            return view

    # --------------------------------------------------------------- drain --
    def begin_step(self, step: int, hyper: AdamHyper, uses: dict[int, int]) -> None:
        self.step, self.hyper = step, hyper
        self.pending_uses = dict(uses)
        self.partial.clear()

    def add_grad(self, c: int, flat: torch.Tensor) -> None:
        """Gradient of one use of chunk c (flat bf16, shard*world elements:
        the chunk's parameters first, zero padding after)."""
        with self._lock:
            if c in self.partial:
                self.partial[c] += flat
            else:
                self.partial[c] = flat
            self.pending_uses[c] -= 1
            if self.pending_uses[c] == 0:
                self._drain(c, self.partial.pop(c))

    def _reduce_peer(self, c: int, grad: torch.Tensor, cur) -> torch.Tensor:
        """exchange="peer": this rank's fp32 reduced shard of chunk c, on cur."""
        s = self.shard[c]
        b = self.n_drains % 2
        self.n_drains += 1
        if self.reduced_free[b] is not None:    # its previous D2H has read it
            cur.wait_event(self.reduced_free[b])
        out = self.reduced[b]
        if self.world == 1:   # the "sum" of one rank: the gradient itself, in fp32
            one = (ctypes.c_void_p * nat.PTK_MAX_PEERS)(grad.data_ptr())
            nat.lib.ptk_peer_reduce_scatter_f32(one, 1, 0, s, vp(out), _sh(cur))
            return out
        if self.sig_reduce is None:
            raise RuntimeError("exchange='peer' needs attach_ipc_peers() before use")
        self.staging[:grad.numel()].copy_(grad)
        self._barrier(self.sig_reduce, cur)      # every rank's gradient is staged
        nat.lib.ptk_peer_reduce_scatter_f32(self.staging_peers, self.world, self.rank, s,
                                            vp(out), _sh(cur))
        self._barrier(self.sig_reduce, cur)      # nobody restages before all have read
        return out

    def _drain(self, c: int, grad: torch.Tensor) -> None:
        s = self.shard[c]
        cur = torch.cuda.current_stream(self.device)
        staged = grad   # already padded to shard*world: reduce-scatter / D2H in place
        peer = self.exchange == "peer"
        if peer:
            reduced = self._reduce_peer(c, grad, cur)
        elif self.comm is not None:
            nat.lib.ptk_chunk_reduce_scatter(self.comm, vp(staged), s, 0, _sh(cur))
        self.d2h.wait_stream(cur)
        src = reduced if peer else staged[self.rank * s:]
        esize = src.element_size()
        landed = []
        if self.timeline is not None:
            self.timeline.gpu(self.d2h, "d2h", "offload_start", f"chunk={c + 1}")
        for lo, n in self._pieces(c):
            nat.lib.ptk_memcpy_d2h_async(vp(self.h_grad[c][lo:]), vp(src[lo:]), esize * n,
                                         _sh(self.d2h))
            ev = torch.cuda.Event()
            ev.record(self.d2h)
            landed.append(ev)
        if peer:
            self.reduced_free[(self.n_drains - 1) % 2] = landed[-1] if landed else None
        else:
            staged.record_stream(self.d2h)
        if self.timeline is not None:
            self.timeline.gpu(self.d2h, "d2h", "offload_end", f"chunk={c + 1}")
        self.counters["d2h_bytes"] += esize * s
        cfg = self.hyper.config(self.step, self.world)
        # the device copy is stale once the host update runs: release the slot
        # (a later fetch into it waits for the compute issued until now)
        if self.resident(c):
            k = self.policy.release(c)
            released = torch.cuda.Event()
            released.record(cur)
            self.slot_released[k] = released
            self.ready.pop(c, None)
        self.piece_done[c] = [threading.Event() for _ in landed]
        self.updates[c] = self.worker.submit(self._host_adam, c, landed, cfg)

    def _host_adam(self, c: int, landed: list, cfg) -> None:
        busy = 0.0
        tl = self.timeline
        for i, ((lo, n), ev, done) in enumerate(zip(self._pieces(c), landed, self.piece_done[c])):
            ev.synchronize()   # this piece's gradients are in host memory
            if i == 0 and tl is not None:
                tl.host("cpu", "update_start", f"chunk={c + 1}")
            t0 = time.perf_counter()
            adam = (nat.raw.ptk_cpu_adam_f32grad if self.exchange == "peer"
                    else nat.raw.ptk_cpu_adam)
            rc = adam(ctypes.byref(cfg), vp(self.h_master[c][lo:]), vp(self.h_m[c][lo:]),
                      vp(self.h_v[c][lo:]), vp(self.h_grad[c][lo:]), vp(self.h_param[c][lo:]), n,
                      self.cpu_threads, None, None)
            busy += time.perf_counter() - t0
            done.set()   # set even on failure: a fetch waiting on it re-raises via result()
            if rc != nat.PTK_OK:
                for d in self.piece_done[c]:
                    d.set()
                raise RuntimeError(f"ptk_cpu_adam: {nat.last_error()}")
        if tl is not None:
            tl.host("cpu", "update_end", f"chunk={c + 1}")
        self.counters["host_adam_s"] = self.counters.get("host_adam_s", 0.0) + busy

    def finish_step(self) -> None:
        for fut in list(self.updates.values()):
            fut.result()

    # ------------------------------------------------- saved-tensor hooks --
    def pack(self, t: torch.Tensor):
        k = self._slot_ptr.get(t.untyped_storage().data_ptr())
        if k is None:
            return ("t", t)
        with self._lock:
            c = self.policy.chunk_in_slot(k)
        return ("ref", c, t.storage_offset(), tuple(t.shape), tuple(t.stride()))

    def unpack(self, packed):
        if packed[0] == "t":
            return packed[1]
        _, c, off, shape, stride = packed
        buf = self.acquire(c, 2 * self.n_total - c, prefetch=c - 1)
        return torch.as_strided(buf, shape, stride, off)


class ChunkGather(torch.autograd.Function):
    """Forward: the parameters of chunk c as views of its gathered buffer.
    Backward: hands this use's gradients of the chunk to the pool, which
    drains the chunk once all uses have reported."""

    @staticmethod
    def forward(ctx, anchor, pool, c, specs, position, prefetch):
        buf = pool.acquire(c, position, prefetch)
        ctx.pool, ctx.c, ctx.specs = pool, c, specs
        outs = []
        for lo, shape in specs:
            n = 1
            for d in shape:
                n *= d
            outs.append(buf[lo:lo + n].view(shape))
        return tuple(outs)

    @staticmethod
    def backward(ctx, *grads):
        pool, c = ctx.pool, ctx.c
        flat = torch.zeros(pool.shard[c] * pool.world, dtype=BF16, device=pool.device)
        for (lo, shape), g in zip(ctx.specs, grads):
            if g is not None:
                flat[lo:lo + g.numel()] = g.reshape(-1)
        pool.add_grad(c, flat)
        return (None,) * 6
