"""Host-side chunk data plane: ZeRO-3 sharded chunk buffers and the per-step
reduce-scatter -> fused Adam -> all-gather over them, driven through the
C-ABI of libptk.so (include/ptk.h). PyTorch is used only to own device memory
and streams.

What this executes is what the reference only models:

* chunk layout: one flat bf16 buffer per chunk of the reference's
  `ChunkLayout` (proj/include/memplan/layout.hpp:27-49); chunk c holds
  `used_bytes / bytes_per_param` parameters in execution order;
* shard mapping: the reference models a rank's shard as
  `floor(used_bytes / w)` bytes (proj/src/cost.cpp:20-22, `shard_bytes`);
  physically the chunk is padded to a multiple of 8*w elements so the shards
  are equal and 16-byte aligned — rank r owns [r*shard, (r+1)*shard);
* persistent chunks hold fp32 master/m/v for the rank's shard on the device
  (the reference's `persistent_chunk_bytes = 8*s_chunk` accounting,
  proj/src/cost.cpp:10, counts the unsharded replica — quirk Q2);
* per step and chunk: reduce-scatter of the bf16 gradient chunk
  (`reduce_time`, proj/src/hardware.cpp:36-38), fused Adam on the owned
  shard with grad scale 1/w (`GpuOptim`, proj/src/sim.cpp:245-250), and
  all-gather of the updated bf16 parameters (`gather_time`,
  proj/src/hardware.cpp:29-34).

Two exchange modes:
  "nccl"  — ptk_chunk_reduce_scatter per chunk, ONE ptk_chunk_adam_table
            launch over every chunk shard, ptk_chunk_allgather per chunk
  "fused" — ptk_fused_step_table: ONE kernel doing RS -> Adam -> AG over
            peer pointers (NVLink P2P on a multi-GPU box) for every chunk,
            bracketed by ptk_peer_barrier. Global-norm clipping / overflow
            skip add a statistics pass (ptk_fused_grad_stats_table) and a
            peer-memory exchange of the 16-byte statistics
            (ptk_stats_publish / ptk_stats_collect) before the update.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import torch

from . import _native as nat

BF16 = torch.bfloat16
F32 = torch.float32

# Seeds of the synthetic state: master = 0.05*u(seed), grads
# = 1e-3*u(seed'), generated over the GLOBAL element index of each chunk so a
# sharded run sees exactly the values of the unsharded run.
MASTER_SCALE = 0.05
GRAD_SCALE = 1e-3


def master_seed(chunk: int) -> int:
    return 1000 * chunk


def grad_seed(chunk: int, rank: int, step: int = 0) -> int:
    return 1000 * chunk + 1 + rank + 100_000 * step


def vp(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else None)


def stream_handle(stream: torch.cuda.Stream | None = None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


@dataclass
class ChunkShard:
    """One chunk as seen by one rank."""

    chunk_id: int
    numel: int        # parameters in the chunk (used_bytes / bytes_per_param)
    world: int
    rank: int
    shard: int        # padded per-rank shard (elements)
    param: torch.Tensor      # bf16[n_pad]  gathered working copy
    grad: torch.Tensor       # bf16[n_pad]  local gradients (RS in place)
    master: torch.Tensor     # fp32[shard]
    exp_avg: torch.Tensor    # fp32[shard]
    exp_avg_sq: torch.Tensor  # fp32[shard]

    @property
    def n_pad(self) -> int:
        return self.shard * self.world

    @property
    def offset(self) -> int:
        return self.rank * self.shard

    def param_shard(self) -> torch.Tensor:
        return self.param[self.offset:self.offset + self.shard]

    def grad_shard(self) -> torch.Tensor:
        return self.grad[self.offset:self.offset + self.shard]

    def owned_numel(self) -> int:
        """Real (unpadded) parameters in this rank's shard."""
        return max(0, min(self.shard, self.numel - self.offset))


@dataclass
class AdamHyper:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    adamw: bool = False
    loss_scale: float = 1.0

    def config(self, step: int, world: int) -> nat.AdamConfig:
        return nat.adam_config(self.lr, self.beta1, self.beta2, self.eps, self.weight_decay,
                               self.adamw, step, 1.0 / (world * self.loss_scale))


class ChunkSet:
    """All persistent chunks of one rank plus the step driver.

    `chunk_numels` comes from a `ChunkLayout` (used_bytes // bytes_per_param
    per chunk). `comm` is a ptk_comm handle (mode "nccl", world > 1);
    `peers` is a list of per-rank ChunkSets (mode "fused" with virtual ranks
    on one device) or a PeerMap of NVLink-mapped pointers.

    `symmetric=True` (mode "nccl" with a communicator): the bf16 param / grad
    chunk buffers come from ncclMemAlloc and are registered as NCCL
    symmetric windows (collective, in chunk order on every rank), so NCCL's
    all-gather / reduce-scatter run their symmetric-memory NVLink kernels;
    `close()` deregisters them (collective: call it on every rank).
    """

    def __init__(self, chunk_numels, world: int = 1, rank: int = 0, device=None,
                 mode: str = "nccl", comm=None, symmetric: bool = False):
        if mode not in ("nccl", "fused"):
            raise ValueError(f"unknown exchange mode {mode!r}")
        if mode == "nccl" and world > 1 and comm is None:
            raise ValueError("world > 1 in nccl mode needs a ptk_comm communicator")
        if symmetric and (mode != "nccl" or comm is None):
            raise ValueError("symmetric windows need mode='nccl' and a ptk_comm communicator")
        self.world, self.rank, self.mode, self.comm = world, rank, mode, comm
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        self.chunks: list[ChunkShard] = []
        self._nccl_mem: list[ctypes.c_void_p] = []    # ncclMemAlloc'd buffers (symmetric)
        self._windows: list[ctypes.c_void_p] = []     # their registered windows

        def flat_bf16(n_pad: int) -> torch.Tensor:
            if not symmetric:
                return torch.zeros(n_pad, dtype=BF16, device=self.device)
            ptr = ctypes.c_void_p()
            with torch.cuda.device(self.device):
                nat.lib.ptk_comm_mem_alloc(ctypes.byref(ptr), 2 * n_pad)
                self._nccl_mem.append(ptr)
                t = _wrap_device(ptr.value, n_pad, self.device).view(BF16)
                t.zero_()
                win = ctypes.c_void_p()
                nat.lib.ptk_comm_window_register(comm, ptr, 2 * n_pad, ctypes.byref(win))
                self._windows.append(win)
            return t

        for c, n in enumerate(chunk_numels):
            shard = nat.shard_elems(int(n), world)
            n_pad = shard * world
            self.chunks.append(ChunkShard(
                c, int(n), world, rank, shard,
                param=flat_bf16(n_pad),
                grad=flat_bf16(n_pad),
                master=torch.zeros(shard, dtype=F32, device=self.device),
                exp_avg=torch.zeros(shard, dtype=F32, device=self.device),
                exp_avg_sq=torch.zeros(shard, dtype=F32, device=self.device)))
        ws_bytes = int(nat.raw.ptk_stats_workspace_bytes())
        self.workspace = torch.zeros(ws_bytes, dtype=torch.uint8, device=self.device)
        self.stats = torch.zeros(2, dtype=torch.float64, device=self.device)  # ptk_grad_stats_t
        self.clip_coef = torch.ones(1, dtype=F32, device=self.device)
        self.skip_flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.step_count = 0
        self.timeline = None         # timeline.Timeline: optim_start/end per chunk
        self.peer_grad_ptrs = None   # fused mode: per chunk (c_void_p * world)
        self.peer_param_ptrs = None
        self.signal_ptrs = None      # fused mode: (c_void_p * world) signal slots
        self.mailbox_ptrs = None     # fused mode: (c_void_p * world) statistics mailboxes
        self.fused_table = None      # ptk_fused_table over every chunk (peers attached)
        self.epoch = 0
        self.stats_epoch = 0
        self.mailbox = (torch.zeros(int(nat.raw.ptk_stats_mailbox_bytes()), dtype=torch.uint8,
                                    device=self.device) if mode == "fused" else None)
        # one ptk_chunk_table over this rank's shards: the step's Adam is ONE launch
        descs = (nat.ChunkDesc * len(self.chunks))()
        for d, c in zip(descs, self.chunks):
            d.master, d.exp_avg, d.exp_avg_sq = (c.master.data_ptr(), c.exp_avg.data_ptr(),
                                                 c.exp_avg_sq.data_ptr())
            d.grad, d.param_out, d.n = c.grad_shard().data_ptr(), c.param_shard().data_ptr(), c.shard
        self.table = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            nat.lib.ptk_chunk_table_create(descs, len(self.chunks), ctypes.byref(self.table))

    def close(self, collective: bool = True) -> None:
        """Releases the native chunk tables (also done on garbage collection)
        and, with `collective` (every rank calls close), the symmetric windows
        and their ncclMemAlloc buffers. Garbage collection never runs the
        collective deregistration (ranks collect at different times): an
        unclosed symmetric set keeps its buffers until the process exits."""
        for name, fn in (("table", "ptk_chunk_table_destroy"),
                         ("fused_table", "ptk_fused_table_destroy")):
            t = getattr(self, name, None)
            if t is not None and t.value:
                getattr(nat.raw, fn)(t)
            setattr(self, name, None)
        if collective and getattr(self, "_nccl_mem", None):
            torch.cuda.synchronize(self.device)
            for c in self.chunks:   # drop the views before the memory goes
                c.param = c.grad = None
            for win in self._windows:
                nat.lib.ptk_comm_window_deregister(self.comm, win)
            for ptr in self._nccl_mem:
                nat.lib.ptk_comm_mem_free(ptr)
            self._windows, self._nccl_mem = [], []

    def __del__(self):
        try:
            self.close(collective=False)
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass

    # ------------------------------------------------------------ sizes --
    @property
    def numel(self) -> int:
        return sum(c.numel for c in self.chunks)

    def algorithmic_hbm_bytes(self) -> int:
        """Per-step HBM bytes of this rank: 28*P/w (Adam) +
        2P(w-1)/w (AG receive) + 2P + 2P/w (RS read local grads, write shard);
        w = 1 -> 28*P. P = real parameters of the chunk."""
        w, tot = self.world, 0
        for c in self.chunks:
            p = c.numel
            tot += 28 * p // w
            if w > 1:
                tot += 2 * p * (w - 1) // w + 2 * p + 2 * p // w
        return tot

    def algorithmic_nvlink_bytes(self) -> int:
        """Per-step NVLink bytes per direction of this rank: 4P(w-1)/w."""
        w = self.world
        return sum(4 * c.numel * (w - 1) // w for c in self.chunks)

    # ---------------------------------------------------- synthetic state --
    def init_synthetic(self, stream=None) -> None:
        """master = 0.05*u(seed_c) over the global index; m = v = 0; the bf16
        working copy of the full chunk is RNE(master) (what an all-gather of
        every rank's shard produces)."""
        s = stream_handle(stream)
        for c in self.chunks:
            nat.lib.ptk_fill_uniform_f32(vp(c.master), c.shard, master_seed(c.chunk_id),
                                         c.offset, MASTER_SCALE, s)
            nat.lib.ptk_fill_uniform_bf16(vp(c.param), c.n_pad, master_seed(c.chunk_id), 0,
                                          MASTER_SCALE, s)
            c.exp_avg.zero_()
            c.exp_avg_sq.zero_()
            self._zero_padding(c)

    def fill_grads(self, step: int = 0, stream=None) -> None:
        """This rank's local gradients of the full chunk: 1e-3*u(seed_{c,rank,step})."""
        s = stream_handle(stream)
        for c in self.chunks:
            nat.lib.ptk_fill_uniform_bf16(vp(c.grad), c.n_pad, grad_seed(c.chunk_id, self.rank, step),
                                          0, GRAD_SCALE, s)
            if c.n_pad > c.numel:
                c.grad[c.numel:].zero_()

    def _zero_padding(self, c: ChunkShard) -> None:
        if c.n_pad > c.numel:
            c.param[c.numel:].zero_()
            lo = max(0, c.numel - c.offset)
            if lo < c.shard:
                c.master[lo:].zero_()

    # --------------------------------------------------------------- step --
    def reset_stats(self, stream=None) -> None:
        nat.lib.ptk_stats_reset(vp(self.stats), stream_handle(stream))

    def step(self, hyper: AdamHyper, stream=None, with_stats: bool = True,
             max_grad_norm: float = 0.0, skip_nonfinite: bool = False) -> None:
        """One optimizer step over every chunk: RS -> Adam -> AG.

        With `max_grad_norm > 0` or `skip_nonfinite`, the global statistics
        of the scaled gradient are needed BEFORE any update. NCCL mode: all
        chunks are reduce-scattered, ptk_grad_stats sums squares / counts
        non-finite elements of every owned shard, the partial statistics are
        all-reduced over the ranks and ptk_clip_coef turns them into a
        device-side clip coefficient and skip flag. Fused mode: a statistics
        pass over the reduced gradient of the owned shards
        (ptk_fused_grad_stats_table), the partials exchanged through the
        peer mailboxes (ptk_stats_publish / ptk_stats_collect, rank-order
        sum: identical on every rank). Either way the update reads both from
        device memory (no host synchronisation anywhere)."""
        self.step_count += 1
        cfg = hyper.config(self.step_count, self.world)
        s = stream_handle(stream)
        stats = vp(self.stats) if with_stats else ctypes.c_void_p(None)
        clip = max_grad_norm > 0 or skip_nonfinite
        if with_stats or clip:
            nat.lib.ptk_stats_reset(vp(self.stats), s)
        if self.mode == "fused":
            self._step_fused(cfg, s, stats, max_grad_norm, skip_nonfinite)
            return
        if clip:
            self._step_clipped(cfg, s, max_grad_norm, skip_nonfinite)
            return
        tl = self.timeline
        if tl is not None:  # per-chunk launches so every chunk's optim span is timed
            for c in self.chunks:
                tl.gpu(stream, "gpu", "optim_start", f"chunk={c.chunk_id + 1}")
                if self.comm is not None:
                    nat.lib.ptk_chunk_reduce_scatter(self.comm, vp(c.grad), c.shard, 0, s)
                nat.lib.ptk_chunk_adam(ctypes.byref(cfg), vp(c.master), vp(c.exp_avg),
                                       vp(c.exp_avg_sq), vp(c.grad_shard()), vp(c.param_shard()),
                                       c.shard, stats, vp(self.workspace), None, None, s)
                if self.comm is not None:
                    nat.lib.ptk_chunk_allgather(self.comm, vp(c.param), c.shard, 0, s)
                tl.gpu(stream, "gpu", "optim_end", f"chunk={c.chunk_id + 1}")
            return
        if self.comm is not None:
            for c in self.chunks:
                nat.lib.ptk_chunk_reduce_scatter(self.comm, vp(c.grad), c.shard, 0, s)
        nat.lib.ptk_chunk_adam_table(ctypes.byref(cfg), self.table, stats, vp(self.workspace),
                                     None, None, s)
        if self.comm is not None:
            for c in self.chunks:
                nat.lib.ptk_chunk_allgather(self.comm, vp(c.param), c.shard, 0, s)

    # ----------------------------------------------- overlapped (per chunk) --
    def begin_overlapped_step(self, hyper: AdamHyper, side: torch.cuda.Stream) -> None:
        """Start a step whose chunks are updated one by one, each as soon as
        its gradients are complete (ChunkedGPT2's backward hooks), on the
        side stream `side` while the backward continues on the compute
        stream. Same kernels and inputs as step(): bit-identical results.

        Fused mode over IPC peers (w > 1): each chunk's REDUCE runs as soon as
        its gradients are complete (ptk_peer_reduce_scatter_f32 between peer
        barriers on the side stream: the NVLink reads overlap the remaining
        backward, as the reference schedules the reduce,
        proj/src/sim.cpp:426-436); after the backward, the Adam of every
        chunk on its fp32 reduced shard (ptk_chunk_adam_f32grad) and the
        all-gather (ptk_peer_allgather). Same fp32 rank-order sums and the
        same update rule as the one-kernel fused step: bit-identical."""
        self._ov_fused = self.mode == "fused" and self.world > 1
        if self._ov_fused and self.signal_ptrs is None:
            raise ValueError("an overlapped fused step needs IPC peers (attach_ipc_peers); "
                             "virtual ranks step together (fused_group_step)")
        if self.mode == "fused" and self.world == 1 and self.fused_table is None:
            raise RuntimeError("fused mode needs peer pointers (attach_virtual_peers)")
        if self._ov_fused and getattr(self, "_reduced", None) is None:
            self._reduced = [torch.empty(c.shard, dtype=F32, device=self.device)
                             for c in self.chunks]
        self.step_count += 1
        self._ov_cfg = hyper.config(self.step_count, self.world)
        self._ov_side = side
        self._ov_done = [False] * len(self.chunks)
        side.wait_stream(torch.cuda.current_stream(self.device))
        nat.lib.ptk_stats_reset(vp(self.stats), stream_handle(side))

    def step_chunk_overlapped(self, ci: int) -> None:
        """RS -> Adam -> AG of chunk ci on the side stream, after everything
        issued so far on the compute stream (its gradient copies)."""
        if self._ov_done[ci]:
            return
        self._ov_done[ci] = True
        side = self._ov_side
        side.wait_stream(torch.cuda.current_stream(self.device))
        s = stream_handle(side)
        c = self.chunks[ci]
        if self._ov_fused:   # the reduce now; update + all-gather after the backward
            self._peer_barrier(s)          # every rank's gradients of chunk ci are final
            nat.lib.ptk_peer_reduce_scatter_f32(self.peer_grad_ptrs[ci], self.world, self.rank,
                                                c.shard, vp(self._reduced[ci]), s)
            self._peer_barrier(s)          # nobody rewrites them before all have read
            return
        tl = self.timeline
        if tl is not None:
            tl.gpu(side, "gpu", "optim_start", f"chunk={c.chunk_id + 1}")
        if self.comm is not None:
            nat.lib.ptk_chunk_reduce_scatter(self.comm, vp(c.grad), c.shard, 0, s)
        nat.lib.ptk_chunk_adam(ctypes.byref(self._ov_cfg), vp(c.master), vp(c.exp_avg),
                               vp(c.exp_avg_sq), vp(c.grad_shard()), vp(c.param_shard()),
                               c.shard, vp(self.stats), vp(self.workspace), None, None, s)
        if self.comm is not None:
            nat.lib.ptk_chunk_allgather(self.comm, vp(c.param), c.shard, 0, s)
        if tl is not None:
            tl.gpu(side, "gpu", "optim_end", f"chunk={c.chunk_id + 1}")

    def finish_overlapped_step(self) -> None:
        """Update the chunks whose hooks never fired (in chunk order), then
        order the compute stream after the side stream."""
        for ci in range(len(self.chunks)):
            self.step_chunk_overlapped(ci)
        if self._ov_fused:
            s = stream_handle(self._ov_side)
            for ci, c in enumerate(self.chunks):
                nat.lib.ptk_chunk_adam_f32grad(ctypes.byref(self._ov_cfg), vp(c.master),
                                               vp(c.exp_avg), vp(c.exp_avg_sq),
                                               vp(self._reduced[ci]), vp(c.param_shard()),
                                               c.shard, vp(self.stats), vp(self.workspace),
                                               None, None, s)
            self._peer_barrier(s)              # every rank's updated shards are written
            for ci, c in enumerate(self.chunks):
                nat.lib.ptk_peer_allgather(self.peer_param_ptrs[ci], self.world, self.rank,
                                           2 * c.shard, s)
            self._peer_barrier(s)              # every rank has pulled every shard
        torch.cuda.current_stream(self.device).wait_stream(self._ov_side)
        self._ov_side = None

    def _peer_barrier(self, s) -> None:
        self.epoch += 1
        nat.lib.ptk_peer_barrier(self.signal_ptrs, self.world, self.rank, self.epoch, s)

    def _step_clipped(self, cfg, s, max_grad_norm: float, skip_nonfinite: bool) -> None:
        for c in self.chunks:
            if self.comm is not None:
                nat.lib.ptk_chunk_reduce_scatter(self.comm, vp(c.grad), c.shard, 0, s)
            nat.lib.ptk_grad_stats(vp(c.grad_shard()), c.shard, ctypes.c_float(cfg.grad_scale),
                                   None, vp(self.stats), vp(self.workspace), s)
        if self.comm is not None:
            nat.lib.ptk_stats_allreduce(self.comm, vp(self.stats), s)
        nat.lib.ptk_clip_coef(vp(self.stats), max_grad_norm, vp(self.clip_coef),
                              vp(self.skip_flag) if skip_nonfinite else None, s)
        nat.lib.ptk_chunk_adam_table(ctypes.byref(cfg), self.table, None, None, vp(self.clip_coef),
                                     vp(self.skip_flag) if skip_nonfinite else None, s)
        if self.comm is not None:
            for c in self.chunks:
                nat.lib.ptk_chunk_allgather(self.comm, vp(c.param), c.shard, 0, s)

    def _step_fused(self, cfg, s, stats, max_grad_norm: float = 0.0,
                    skip_nonfinite: bool = False) -> None:
        if self.fused_table is None:
            raise RuntimeError("fused mode needs peer pointers (attach_virtual_peers / attach_ipc_peers)")
        clip = max_grad_norm > 0 or skip_nonfinite
        if clip and self.signal_ptrs is None and self.world > 1:
            raise ValueError("virtual ranks share one stream: a clipped fused step must be issued "
                             "for all of them together (fused_group_step)")
        if self.signal_ptrs is not None:
            self.epoch += 1
            nat.lib.ptk_peer_barrier(self.signal_ptrs, self.world, self.rank, self.epoch, s)
        if clip:
            self._fused_stats_phase(cfg, s)
            self._fused_publish(s)
            self._fused_collect(s, max_grad_norm, skip_nonfinite)
            self._fused_update(cfg, s, None, clip=True, skip=skip_nonfinite)
        else:
            self._fused_update(cfg, s, stats)
        if self.signal_ptrs is not None:
            self.epoch += 1
            nat.lib.ptk_peer_barrier(self.signal_ptrs, self.world, self.rank, self.epoch, s)

    # The phases of a fused step (fused_group_step issues them rank by rank
    # for virtual ranks sharing one stream).
    def _fused_stats_phase(self, cfg, s) -> None:
        nat.lib.ptk_fused_grad_stats_table(ctypes.byref(cfg), self.fused_table, vp(self.stats),
                                           vp(self.workspace), s)

    def _fused_publish(self, s) -> None:
        self.stats_epoch += 1
        nat.lib.ptk_stats_publish(vp(self.stats), self.mailbox_ptrs, self.world, self.rank,
                                  self.stats_epoch, s)

    def _fused_collect(self, s, max_grad_norm: float, skip_nonfinite: bool) -> None:
        nat.lib.ptk_stats_collect(vp(self.mailbox), self.world, self.stats_epoch, max_grad_norm,
                                  vp(self.stats), vp(self.clip_coef),
                                  vp(self.skip_flag) if skip_nonfinite else None, s)

    def _fused_update(self, cfg, s, stats, clip: bool = False, skip: bool = False) -> None:
        nat.lib.ptk_fused_step_table(ctypes.byref(cfg), self.fused_table, stats,
                                     vp(self.workspace), vp(self.clip_coef) if clip else None,
                                     vp(self.skip_flag) if skip else None, s)

    def _build_fused_table(self, kernel: int) -> None:
        if self.fused_table is not None:
            nat.raw.ptk_fused_table_destroy(self.fused_table)
        descs = (nat.FusedDesc * len(self.chunks))()
        for d, c, gp, pp in zip(descs, self.chunks, self.peer_grad_ptrs, self.peer_param_ptrs):
            for r in range(self.world):
                d.grad_peers[r], d.param_peers[r] = gp[r], pp[r]
            d.master, d.exp_avg, d.exp_avg_sq = (c.master.data_ptr(), c.exp_avg.data_ptr(),
                                                 c.exp_avg_sq.data_ptr())
            d.shard = c.shard
        self.fused_table = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            nat.lib.ptk_fused_table_create(descs, len(self.chunks), self.world, self.rank, kernel,
                                           ctypes.byref(self.fused_table))

    @property
    def fused_kernel(self) -> str:
        """'tma' or 'ldg': the fused kernel this rank's table runs."""
        k = int(nat.raw.ptk_fused_table_kernel(self.fused_table)) if self.fused_table else -1
        return {nat.PTK_FUSED_TMA: "tma", nat.PTK_FUSED_LDG: "ldg"}.get(k, "none")

    def attach_virtual_peers(self, sets: list["ChunkSet"]) -> None:
        """Single-GPU validation of the fused path: `sets[r]` plays rank r.
        The kernel then reads every virtual rank's gradient buffer and writes
        every virtual rank's parameter buffer exactly as it would over NVLink."""
        arr = ctypes.c_void_p * PTK_MAX
        self.peer_grad_ptrs, self.peer_param_ptrs = [], []
        for ci in range(len(self.chunks)):
            g = arr(*[sets[r].chunks[ci].grad.data_ptr() for r in range(self.world)])
            p = arr(*[sets[r].chunks[ci].param.data_ptr() for r in range(self.world)])
            self.peer_grad_ptrs.append(g)
            self.peer_param_ptrs.append(p)
        self.mailbox_ptrs = arr(*[sets[r].mailbox.data_ptr() for r in range(self.world)])
        # every buffer is on this device: the TMA ring (PTK_FUSED_KERNEL may force one)
        self._build_fused_table(fused_kernel_choice(same_device=True))

    def attach_ipc_peers(self, group=None) -> None:
        """Multi-GPU fused mode: map every peer's gradient / parameter chunk
        buffers and signal slots into this process over NVLink (cudaIpc
        handles exchanged through torch.distributed, which is only plumbing
        here). Must be called collectively by all ranks."""
        import torch.distributed as dist
        arr = ctypes.c_void_p * PTK_MAX
        self.signal = torch.zeros(PTK_MAX, dtype=torch.int32, device=self.device)
        bufs = ([c.grad for c in self.chunks] + [c.param for c in self.chunks] +
                [self.signal, self.mailbox])
        # ptrs[r][k]: rank r's k-th buffer as mapped here
        ptrs, self._opened, same_device = map_peer_buffers(bufs, self.world, self.rank,
                                                           self.device, group)
        n = len(self.chunks)
        self.peer_grad_ptrs = [arr(*[ptrs[r][ci] for r in range(self.world)]) for ci in range(n)]
        self.peer_param_ptrs = [arr(*[ptrs[r][n + ci] for r in range(self.world)])
                                for ci in range(n)]
        self.signal_ptrs = arr(*[ptrs[r][2 * n] for r in range(self.world)])
        self.mailbox_ptrs = arr(*[ptrs[r][2 * n + 1] for r in range(self.world)])
        self.epoch = 0
        self.stats_epoch = 0
        self._build_fused_table(fused_kernel_choice(same_device))
        dist.barrier(group=group)

    def close_ipc_peers(self) -> None:
        for base in getattr(self, "_opened", []):
            nat.lib.ptk_ipc_close_handle(base)
        self._opened = []

    def grad_stats(self) -> tuple[float, int]:
        v = self.stats.cpu()
        sumsq = float(v[0])
        nonfinite = int(v.view(torch.int64)[1])
        return sumsq, nonfinite


PTK_MAX = nat.PTK_MAX_PEERS


def map_peer_buffers(bufs: list[torch.Tensor], world: int, rank: int, device, group=None):
    """Collective: every rank's `bufs` mapped into this process through cudaIpc
    handles (exchanged over torch.distributed -- plumbing only). Returns
    (ptrs, opened, same_device): ptrs[r][k] = rank r's k-th buffer as seen
    here, the opened mappings (for ptk_ipc_close_handle), and whether every
    rank is on this physical GPU (by UUID, not ordinal: ranks may be isolated
    with CUDA_VISIBLE_DEVICES)."""
    import torch.distributed as dist
    mine = []
    for t in bufs:
        h = (ctypes.c_uint8 * nat.PTK_IPC_HANDLE_BYTES)()
        off = ctypes.c_int64()
        nat.lib.ptk_ipc_get_handle(vp(t), h, ctypes.byref(off))
        mine.append((bytes(h), off.value))
    torch.cuda.synchronize(device)
    uuid = str(torch.cuda.get_device_properties(device).uuid)
    everyone = [None] * world
    dist.all_gather_object(everyone, (uuid, mine), group=group)
    same_device = all(u == uuid for u, _ in everyone)
    opened, ptrs = [], []
    for r, (_, handles) in enumerate(everyone):
        row = []
        for k, (hb, off) in enumerate(handles):
            if r == rank:
                row.append(bufs[k].data_ptr())
                continue
            base = ctypes.c_void_p()
            nat.lib.ptk_ipc_open_handle((ctypes.c_uint8 * len(hb)).from_buffer_copy(hb),
                                        ctypes.byref(base))
            opened.append(base)
            row.append(base.value + off)
        ptrs.append(row)
    return ptrs, opened, same_device


class _CudaArray:
    """A raw device range seen through __cuda_array_interface__ (no ownership)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i2", "data": (ptr, False),
                                         "strides": None, "version": 3}


def _wrap_device(ptr: int, n: int, device: torch.device) -> torch.Tensor:
    """int16 tensor view of n elements at device pointer `ptr` (memory owned elsewhere)."""
    return torch.as_tensor(_CudaArray(ptr, n), device=device)


def fused_kernel_choice(same_device: bool) -> int:
    """The fused kernel for a peer table: PTK_FUSED_KERNEL=tma|ldg if set,
    else the TMA ring (dynamic tile schedule, 1.03-1.05 of the measured HBM
    peak with virtual ranks) wherever the peer buffers live -- bulk copies
    address cudaIpc / peer mappings like any global memory. The
    register-staged kernel (plain 128-bit peer loads / stores) stays
    selectable. Chosen once per table."""
    env = os.environ.get("PTK_FUSED_KERNEL", "")
    if env == "ldg":
        return nat.PTK_FUSED_LDG
    return nat.PTK_FUSED_TMA


def fused_group_step(sets: list[ChunkSet], hyper: AdamHyper, stream=None, with_stats: bool = True,
                     max_grad_norm: float = 0.0, skip_nonfinite: bool = False) -> None:
    """One fused step of W VIRTUAL ranks sharing a device and a stream
    (single-GPU validation of the N>1 path): without clipping, each rank's
    fused launch in turn; with clipping / overflow skip, every rank's
    statistics pass, then every publish, every collect, every update -- the
    order the peer mailboxes need when the ranks cannot run concurrently."""
    clip = max_grad_norm > 0 or skip_nonfinite
    if not clip:
        for cs in sets:
            cs.step(hyper, stream=stream, with_stats=with_stats)
        return
    s = stream_handle(stream)
    cfgs = []
    for cs in sets:
        if cs.fused_table is None or cs.signal_ptrs is not None:
            raise ValueError("fused_group_step drives virtual ranks (attach_virtual_peers)")
        cs.step_count += 1
        cfgs.append(hyper.config(cs.step_count, cs.world))
        nat.lib.ptk_stats_reset(vp(cs.stats), s)
    for cs, cfg in zip(sets, cfgs):
        cs._fused_stats_phase(cfg, s)
    for cs in sets:
        cs._fused_publish(s)
    for cs in sets:
        cs._fused_collect(s, max_grad_norm, skip_nonfinite)
    for cs, cfg in zip(sets, cfgs):
        cs._fused_update(cfg, s, None, clip=True, skip=skip_nonfinite)
