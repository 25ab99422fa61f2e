"""ctypes access to the CPU oracle (oracle/_ref/liboracle_chunk.so).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline arm import this module. The oracle is the checker, never the thing
measured for the GPU arm or shipped.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_double, c_float, c_int, c_int64, c_uint16, c_uint64
from ctypes import c_void_p

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(REPO, "oracle", "_ref", "liboracle_chunk.so")


class OracleScalars(Structure):
    _fields_ = [(n, c_float) for n in ("gscale", "wd", "decay", "w1", "b2", "w2", "eps",
                                       "neg_step_size", "bc2_sqrt")] + [("adamw", c_int)]


def _load():
    if not os.path.exists(ORACLE_SO):
        raise ImportError(f"{ORACLE_SO} missing: run `make -C oracle port`")
    lib = ctypes.CDLL(ORACLE_SO)
    lib.oracle_adam_scalars.argtypes = [c_double, c_double, c_double, c_double, c_double, c_int,
                                        c_int, c_double, POINTER(OracleScalars)]
    for name in ("oracle_adam_step", "oracle_adam_step_f32grad"):
        getattr(lib, name).argtypes = [POINTER(OracleScalars), c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_int64, POINTER(c_double),
                                       POINTER(c_int64)]
    lib.oracle_shard_elems.restype = c_int64
    lib.oracle_shard_elems.argtypes = [c_int64, c_int]
    lib.oracle_allgather_bf16.argtypes = [POINTER(c_void_p), c_int, c_int64, c_void_p]
    lib.oracle_reduce_scatter_bf16.argtypes = [POINTER(c_void_p), c_int, c_int, c_int64, c_void_p]
    lib.oracle_reduce_scatter_f32.argtypes = [POINTER(c_void_p), c_int, c_int, c_int64, c_void_p]
    lib.oracle_f32_to_bf16.restype = c_uint16
    lib.oracle_f32_to_bf16.argtypes = [c_float]
    lib.oracle_bf16_to_f32.restype = c_float
    lib.oracle_bf16_to_f32.argtypes = [c_uint16]
    lib.oracle_fill_uniform_f32.argtypes = [c_void_p, c_int64, c_uint64, c_int64, c_float]
    lib.oracle_fill_uniform_bf16.argtypes = [c_void_p, c_int64, c_uint64, c_int64, c_float]
    lib.oracle_num_threads.restype = c_int
    lib.oracle_set_num_threads.argtypes = [c_int]
    return lib


lib = _load()


def _p(a: np.ndarray) -> c_void_p:
    assert a.flags["C_CONTIGUOUS"]
    return c_void_p(a.ctypes.data)


def scalars(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, adamw=False, step=1,
            grad_scale=1.0) -> OracleScalars:
    s = OracleScalars()
    lib.oracle_adam_scalars(lr, beta1, beta2, eps, weight_decay, int(bool(adamw)), int(step),
                            grad_scale, ctypes.byref(s))
    return s


def adam_step(s: OracleScalars, master, m, v, grad, param_out=None):
    """In place on numpy arrays; grad uint16 (bf16 bits) or float32. Returns
    (sumsq, nonfinite)."""
    sq, bad = c_double(0.0), c_int64(0)
    fn = lib.oracle_adam_step if grad.dtype == np.uint16 else lib.oracle_adam_step_f32grad
    fn(ctypes.byref(s), _p(master), _p(m), _p(v), _p(grad),
       _p(param_out) if param_out is not None else c_void_p(None), master.size,
       ctypes.byref(sq), ctypes.byref(bad))
    return sq.value, bad.value


def shard_elems(n: int, world: int) -> int:
    return int(lib.oracle_shard_elems(n, world))


def reduce_scatter(grads: list[np.ndarray], rank: int, shard: int, fp32: bool = False):
    arr = (c_void_p * len(grads))(*[g.ctypes.data for g in grads])
    if fp32:
        out = np.empty(shard, dtype=np.float32)
        lib.oracle_reduce_scatter_f32(arr, len(grads), rank, shard, _p(out))
    else:
        out = np.empty(shard, dtype=np.uint16)
        lib.oracle_reduce_scatter_bf16(arr, len(grads), rank, shard, _p(out))
    return out


def allgather(shards: list[np.ndarray]) -> np.ndarray:
    shard = shards[0].size
    out = np.empty(shard * len(shards), dtype=np.uint16)
    arr = (c_void_p * len(shards))(*[s.ctypes.data for s in shards])
    lib.oracle_allgather_bf16(arr, len(shards), shard, _p(out))
    return out


def fill_f32(n: int, seed: int, scale: float, index0: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    lib.oracle_fill_uniform_f32(_p(out), n, seed, index0, scale)
    return out


def fill_bf16(n: int, seed: int, scale: float, index0: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.uint16)
    lib.oracle_fill_uniform_bf16(_p(out), n, seed, index0, scale)
    return out


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = 0x7FFF
    return r


def num_threads() -> int:
    return int(lib.oracle_num_threads())


def set_num_threads(n: int) -> None:
    lib.oracle_set_num_threads(int(n))
