"""ctypes binding of libptk.so (include/ptk.h) — the only way Python reaches the
B200 data plane. There is deliberately NO fallback: if the shared library is
missing or fails to load, importing this module raises, so a GPU run can never
silently route through a CPU or eager-PyTorch path.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_char_p, c_double, c_float, c_int32, c_int64, c_size_t
from ctypes import c_uint8, c_uint64, c_ulonglong, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libptk.so")

PTK_OK = 0
PTK_EINVAL, PTK_ECUDA, PTK_ENCCL, PTK_EUNSUPPORTED = -1, -2, -3, -4   # include/ptk.h
PTK_MAX_PEERS = 8
PTK_UNIQUE_ID_BYTES = 128
PTK_IPC_HANDLE_BYTES = 64


class PtkError(RuntimeError):
    """A libptk call returned a nonzero status (message from ptk_last_error)."""


class AdamConfig(Structure):
    _fields_ = [
        ("lr", c_double),
        ("beta1", c_double),
        ("beta2", c_double),
        ("eps", c_double),
        ("weight_decay", c_double),
        ("adamw", c_int32),
        ("step", c_int32),
        ("grad_scale", c_double),
    ]


class AdamScalars(Structure):
    _fields_ = [(n, c_float) for n in ("gscale", "wd", "decay", "w1", "b2", "w2", "eps",
                                       "neg_step_size", "bc2_sqrt")] + [("adamw", c_int32)]


class GradStats(Structure):
    _fields_ = [("sumsq", c_double), ("nonfinite", c_ulonglong)]


class ChunkDesc(Structure):
    """ptk_chunk_desc: one chunk shard of a ptk_chunk_table."""
    _fields_ = [("master", c_void_p), ("exp_avg", c_void_p), ("exp_avg_sq", c_void_p),
                ("grad", c_void_p), ("param_out", c_void_p), ("n", c_int64)]


class FusedDesc(Structure):
    """ptk_fused_desc: one chunk of a ptk_fused_table (every rank's buffers)."""
    _fields_ = [("grad_peers", c_void_p * PTK_MAX_PEERS), ("param_peers", c_void_p * PTK_MAX_PEERS),
                ("master", c_void_p), ("exp_avg", c_void_p), ("exp_avg_sq", c_void_p),
                ("shard", c_int64)]


PTK_FUSED_AUTO, PTK_FUSED_TMA, PTK_FUSED_LDG = 0, 1, 2


# name -> (restype, argtypes); int-returning functions are status-checked.
_SIGNATURES = {
    "ptk_last_error": (c_char_p, []),
    "ptk_version": (c_char_p, []),
    "ptk_adam_derive": (c_int32, [POINTER(AdamConfig), POINTER(AdamScalars)]),
    "ptk_shard_elems": (c_int64, [c_int64, c_int32]),
    "ptk_stats_workspace_bytes": (c_int64, []),
    "ptk_adam_kernel_name": (c_char_p, []),
    "ptk_fused_kernel_name": (c_char_p, []),
    "ptk_profile_host_memory_bw": (c_int32, [c_int64, c_int32, c_double, POINTER(c_double)]),
    "ptk_chunk_adam": (c_int32, [POINTER(AdamConfig), c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p]),
    "ptk_chunk_adam_f32grad": (c_int32, [POINTER(AdamConfig), c_void_p, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p]),
    "ptk_grad_stats": (c_int32, [c_void_p, c_int64, c_float, c_void_p, c_void_p, c_void_p,
                                 c_void_p]),
    "ptk_grad_prep": (c_int32, [c_void_p, c_int64, c_float, c_void_p, c_void_p, c_void_p,
                                c_void_p]),
    "ptk_stats_reset": (c_int32, [c_void_p, c_void_p]),
    "ptk_clip_coef": (c_int32, [c_void_p, c_double, c_void_p, c_void_p, c_void_p]),
    "ptk_fused_rs_adam_ag": (c_int32, [POINTER(AdamConfig), POINTER(c_void_p), POINTER(c_void_p),
                                       c_int32, c_int32, c_int64, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_void_p]),
    "ptk_chunk_table_create": (c_int32, [POINTER(ChunkDesc), c_int32, POINTER(c_void_p)]),
    "ptk_chunk_table_destroy": (c_int32, [c_void_p]),
    "ptk_chunk_table_params": (c_int64, [c_void_p]),
    "ptk_chunk_adam_table": (c_int32, [POINTER(AdamConfig), c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_void_p]),
    "ptk_fused_table_create": (c_int32, [POINTER(FusedDesc), c_int32, c_int32, c_int32, c_int32,
                                         POINTER(c_void_p)]),
    "ptk_fused_table_destroy": (c_int32, [c_void_p]),
    "ptk_fused_table_kernel": (c_int32, [c_void_p]),
    "ptk_fused_step_table": (c_int32, [POINTER(AdamConfig), c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_void_p]),
    "ptk_fused_grad_stats_table": (c_int32, [POINTER(AdamConfig), c_void_p, c_void_p, c_void_p,
                                             c_void_p]),
    "ptk_stats_mailbox_bytes": (c_int64, []),
    "ptk_stats_publish": (c_int32, [c_void_p, POINTER(c_void_p), c_int32, c_int32, c_int32,
                                    c_void_p]),
    "ptk_stats_collect": (c_int32, [c_void_p, c_int32, c_int32, c_double, c_void_p, c_void_p,
                                    c_void_p, c_void_p]),
    "ptk_fill_uniform_f32": (c_int32, [c_void_p, c_int64, c_uint64, c_int64, c_float, c_void_p]),
    "ptk_fill_uniform_bf16": (c_int32, [c_void_p, c_int64, c_uint64, c_int64, c_float, c_void_p]),
    "ptk_busy_wait": (c_int32, [c_int64, c_void_p]),
    "ptk_comm_unique_id": (c_int32, [POINTER(c_uint8)]),
    "ptk_comm_init": (c_int32, [POINTER(c_void_p), c_int32, c_int32, POINTER(c_uint8)]),
    "ptk_comm_destroy": (c_int32, [c_void_p]),
    "ptk_chunk_allgather": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p]),
    "ptk_chunk_reduce_scatter": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p]),
    "ptk_comm_barrier": (c_int32, [c_void_p, c_void_p]),
    "ptk_stats_allreduce": (c_int32, [c_void_p, c_void_p, c_void_p]),
    "ptk_comm_wait": (c_int32, [c_void_p, c_void_p, c_int64]),
    "ptk_comm_async_error": (c_int32, [c_void_p]),
    "ptk_comm_abort": (c_int32, [c_void_p]),
    "ptk_comm_mem_alloc": (c_int32, [POINTER(c_void_p), c_int64]),
    "ptk_comm_mem_free": (c_int32, [c_void_p]),
    "ptk_comm_window_register": (c_int32, [c_void_p, c_void_p, c_int64, POINTER(c_void_p)]),
    "ptk_comm_window_deregister": (c_int32, [c_void_p, c_void_p]),
    "ptk_ipc_get_handle": (c_int32, [c_void_p, POINTER(c_uint8), POINTER(c_int64)]),
    "ptk_ipc_open_handle": (c_int32, [POINTER(c_uint8), POINTER(c_void_p)]),
    "ptk_ipc_close_handle": (c_int32, [c_void_p]),
    "ptk_peer_barrier": (c_int32, [POINTER(c_void_p), c_int32, c_int32, c_int32, c_void_p]),
    "ptk_host_alloc_pinned": (c_int32, [POINTER(c_void_p), c_size_t]),
    "ptk_host_free_pinned": (c_int32, [c_void_p]),
    "ptk_memcpy_h2d_async": (c_int32, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "ptk_memcpy_d2h_async": (c_int32, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "ptk_cpu_adam": (c_int32, [POINTER(AdamConfig), c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_int64, c_int32, POINTER(c_double), POINTER(c_int64)]),
    "ptk_cpu_adam_f32grad": (c_int32, [POINTER(AdamConfig), c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_int64, c_int32, POINTER(c_double),
                                       POINTER(c_int64)]),
    "ptk_peer_reduce_scatter_f32": (c_int32, [POINTER(c_void_p), c_int32, c_int32, c_int64,
                                              c_void_p, c_void_p]),
    "ptk_peer_allgather": (c_int32, [POINTER(c_void_p), c_int32, c_int32, c_int64, c_void_p]),
    "ptk_execute_plan": (c_int32, [c_char_p, c_char_p, c_char_p, c_void_p, c_int32, c_double,
                                   c_int32, c_char_p, c_char_p]),
    "ptk_measure_profile": (c_int32, [c_char_p, c_void_p, c_int32, c_char_p]),
    "ptk_profile_copy_bw": (c_int32, [c_int64, POINTER(c_double), POINTER(c_double)]),
    "ptk_profile_collective": (c_int32, [c_void_p, c_int32, c_int64, POINTER(c_double),
                                         POINTER(c_double)]),
    "ptk_profile_gpu_adam_rate": (c_int32, [c_int64, POINTER(c_double)]),
    "ptk_profile_cpu_adam_rate": (c_int32, [c_int64, POINTER(c_double)]),
    "ptk_stream_create": (c_int32, [POINTER(c_void_p), c_int32]),
    "ptk_stream_destroy": (c_int32, [c_void_p]),
    "ptk_event_create": (c_int32, [POINTER(c_void_p)]),
    "ptk_event_destroy": (c_int32, [c_void_p]),
    "ptk_event_record": (c_int32, [c_void_p, c_void_p]),
    "ptk_stream_wait_event": (c_int32, [c_void_p, c_void_p]),
    "ptk_event_elapsed_ms": (c_int32, [c_void_p, c_void_p, POINTER(c_float)]),
    "ptk_stream_synchronize": (c_int32, [c_void_p]),
    "ptk_device_synchronize": (c_int32, []),
    "ptk_kernel_launch_count": (c_int64, []),
    "ptk_pool_create": (c_int32, [c_int32, c_int32, c_int32, POINTER(c_void_p)]),
    "ptk_pool_destroy": (None, [c_void_p]),
    "ptk_pool_grant": (c_int32, [c_void_p, c_int32, c_int32, POINTER(c_int32), c_int32, c_int32,
                                 POINTER(c_int32), POINTER(c_int32)]),
    "ptk_pool_arrived": (c_int32, [c_void_p, c_int32]),
    "ptk_pool_release": (c_int32, [c_void_p, c_int32, POINTER(c_int32)]),
    "ptk_pool_slot_of": (c_int32, [c_void_p, c_int32]),
    "ptk_pool_chunk_in_slot": (c_int32, [c_void_p, c_int32]),
    "ptk_pool_residency": (c_int32, [c_void_p, c_int32]),
    "ptk_memplan_run": (c_int32, [c_int32, POINTER(c_char_p), POINTER(c_void_p),
                                  POINTER(c_void_p)]),
    "ptk_free": (None, [c_void_p]),
}
# int32-returning functions whose result is a value, not a status
_VALUE_RESULTS = {"ptk_pool_slot_of", "ptk_pool_chunk_in_slot", "ptk_pool_residency",
                  "ptk_memplan_run"}

EXPORTED_SYMBOLS = tuple(_SIGNATURES)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libptk.so not found at {LIB_PATH}: build it with `make ptk` (or "
        "`python -c 'import __graft_entry__ as g; g.build()'`). There is no fallback path.")

# libptk.so and torch both need `libnccl.so.2`; whichever loads first binds
# the soname for the process. torch's bundled NCCL (2.28) is a superset of the
# system one (2.27) that libptk was linked against, so torch goes first: with
# libptk first, importing torch later fails (libtorch_cuda: undefined symbol
# ncclDevCommCreate).
import torch  # noqa: E402,F401

_lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
for _name, (_res, _args) in _SIGNATURES.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def last_error() -> str:
    msg = _lib.ptk_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str) -> None:
    if rc != PTK_OK:
        raise PtkError(f"{what} failed ({rc}): {last_error()}")


class _Lib:
    """Status-checked attribute access: lib.ptk_chunk_adam(...) raises on error."""

    def __getattr__(self, name):
        fn = getattr(_lib, name)
        if _SIGNATURES[name][0] is c_int32 and name not in _VALUE_RESULTS:
            def call(*args, _fn=fn, _name=name):
                rc = _fn(*args)
                check(rc, _name)
                return rc
            return call
        return fn


lib = _Lib()
raw = _lib


def adam_config(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, adamw=False,
                step=1, grad_scale=1.0) -> AdamConfig:
    return AdamConfig(lr, beta1, beta2, eps, weight_decay, int(bool(adamw)), int(step),
                      float(grad_scale))


def derive_scalars(cfg: AdamConfig) -> AdamScalars:
    out = AdamScalars()
    lib.ptk_adam_derive(ctypes.byref(cfg), ctypes.byref(out))
    return out


def shard_elems(n: int, world: int) -> int:
    return int(_lib.ptk_shard_elems(n, world))


def launch_count() -> int:
    return int(_lib.ptk_kernel_launch_count())


class BufferPool:
    """The runtime's chunk residency policy (memplan::ChunkBufferPool through
    ptk_pool_*): slot grants, farthest-next-use eviction, arrival and release.
    Chunk ids are 0-based here (1-based in C); positions are the C ones
    (forward of 0-based chunk c = c + 1, backward = 2N - c)."""

    def __init__(self, n_chunk: int, n_persist: int, n_buffer: int):
        h = c_void_p()
        lib.ptk_pool_create(n_chunk, n_persist, n_buffer, ctypes.byref(h))
        self._h = h
        self.n_chunk, self.n_persist, self.n_buffer = n_chunk, n_persist, n_buffer

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.ptk_pool_destroy(self._h)
            self._h = None

    def grant(self, c: int, now: int, pinned=(), demand: bool = False
              ) -> tuple[int, int | None] | None:
        """(slot, evicted 0-based chunk or None), or None when no slot can be
        granted for c at position `now` (demand: c is needed right now)."""
        pin = (c_int32 * max(1, len(pinned)))(*[p + 1 for p in pinned])
        slot, ev = c_int32(), c_int32()
        lib.ptk_pool_grant(self._h, c + 1, now, pin, len(pinned), int(demand),
                           ctypes.byref(slot), ctypes.byref(ev))
        if slot.value < 0:
            return None
        return slot.value, (ev.value - 1 if ev.value else None)

    def arrived(self, c: int) -> None:
        lib.ptk_pool_arrived(self._h, c + 1)

    def release(self, c: int) -> int:
        slot = c_int32()
        lib.ptk_pool_release(self._h, c + 1, ctypes.byref(slot))
        return slot.value

    def slot_of(self, c: int) -> int:
        return int(_lib.ptk_pool_slot_of(self._h, c + 1))

    def chunk_in_slot(self, s: int) -> int | None:
        c = int(_lib.ptk_pool_chunk_in_slot(self._h, s))
        return c - 1 if c else None

    def residency(self, c: int) -> int:
        return int(_lib.ptk_pool_residency(self._h, c + 1))


def memplan_run(args: list[str]) -> tuple[int, str, str]:
    """The planner CLI in process (ptk_memplan_run): (exit code, stdout, stderr)."""
    argv = (c_char_p * max(1, len(args)))(*[a.encode() for a in args])
    out, err = c_void_p(), c_void_p()
    rc = int(_lib.ptk_memplan_run(len(args), argv, ctypes.byref(out), ctypes.byref(err)))
    try:
        so = ctypes.string_at(out).decode() if out.value else ""
        se = ctypes.string_at(err).decode() if err.value else ""
    finally:
        _lib.ptk_free(out)
        _lib.ptk_free(err)
    return rc, so, se
