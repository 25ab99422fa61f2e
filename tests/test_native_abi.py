"""The C-ABI library loads without a GPU, exports every entry point that
include/ptk.h declares, and its host-only functions (scalar derivation, shard
mapping, K6 host Adam) agree bit-exactly with the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle_lib as ol

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    text = open(os.path.join(REPO, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ptk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2406_08334_b200 import _native as nat
    names = _declared("ptk.h")
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(nat.raw, n)]
    assert not missing, missing
    # and the Python binding declares a signature for each of them
    assert set(names) == set(nat.EXPORTED_SYMBOLS)


def test_symbols_visible_to_dlsym():
    lib = ctypes.CDLL(os.path.join(REPO, "paper_2406_08334_b200", "libptk.so"))
    for n in _declared("ptk.h"):
        getattr(lib, n)


@pytest.mark.parametrize("cfg", [dict(step=1), dict(step=7, adamw=True, weight_decay=0.1),
                                 dict(step=3, weight_decay=0.01, grad_scale=0.125, lr=3e-4)])
def test_scalar_derivation_matches_oracle(cfg):
    from paper_2406_08334_b200 import _native as nat
    a = nat.derive_scalars(nat.adam_config(**cfg))
    b = ol.scalars(**cfg)
    for f, _ in nat.AdamScalars._fields_:
        assert getattr(a, f) == getattr(b, f), f


@pytest.mark.parametrize("n,w", [(0, 1), (1, 1), (1001, 2), (1001, 8), (512_420_800, 8),
                                 (201_379_840, 3)])
def test_shard_mapping(n, w):
    from paper_2406_08334_b200 import _native as nat
    assert nat.shard_elems(n, w) == ol.shard_elems(n, w)


def test_host_adam_k6_bit_exact():
    from paper_2406_08334_b200 import _native as nat
    n = 200_003
    master = ol.fill_f32(n, 0, 0.05)
    g = ol.fill_bf16(n, 1, 1e-3)
    a = [master.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)]
    b = [master.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)]
    pa = np.zeros(n, np.uint16)
    pb = np.zeros(n, np.uint16)
    for step in (1, 2, 3):
        cfg = nat.adam_config(step=step, weight_decay=0.01, adamw=True, grad_scale=0.5)
        sq, bad = ctypes.c_double(), ctypes.c_int64()
        nat.lib.ptk_cpu_adam(ctypes.byref(cfg), *[ctypes.c_void_p(x.ctypes.data) for x in a],
                             ctypes.c_void_p(g.ctypes.data), ctypes.c_void_p(pa.ctypes.data), n,
                             0, ctypes.byref(sq), ctypes.byref(bad))
        osq, obad = ol.adam_step(ol.scalars(step=step, weight_decay=0.01, adamw=True,
                                            grad_scale=0.5), *b, g, pb)
        assert bad.value == obad == 0
        assert abs(sq.value - osq) <= 1e-9 * osq
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x.view(np.uint32), y.view(np.uint32))
    np.testing.assert_array_equal(pa, pb)


@pytest.mark.parametrize("mode", ["adam", "adamw", "l2"])
@pytest.mark.parametrize("offset", [0, 1, 5])
def test_host_adam_all_modes_unaligned_bit_exact(mode, offset):
    """Every update rule of the host Adam (incl. the AVX-512 non-temporal
    output path) at unaligned output addresses, with a NaN and infinities in
    the gradients: bit-identical to the oracle, bf16 rounding included."""
    from paper_2406_08334_b200 import _native as nat
    n = 70_001
    wd, adamw = {"adam": (0.0, False), "adamw": (0.01, True), "l2": (0.01, False)}[mode]
    master = ol.fill_f32(n, 3, 0.05)
    g = ol.fill_bf16(n, 4, 1e-3)
    g[17] = 0x7fc0   # NaN
    g[18] = 0x7f80   # +inf
    g[n - 3] = 0xff80  # -inf
    a = [master.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)]
    b = [master.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)]
    buf = np.zeros(n + 8, np.uint16)
    pa = buf[offset:offset + n]
    pb = np.zeros(n, np.uint16)
    for step in (1, 2):
        cfg = nat.adam_config(step=step, weight_decay=wd, adamw=adamw, grad_scale=0.5)
        nat.lib.ptk_cpu_adam(ctypes.byref(cfg), *[ctypes.c_void_p(x.ctypes.data) for x in a],
                             ctypes.c_void_p(g.ctypes.data), ctypes.c_void_p(pa.ctypes.data), n,
                             3, None, None)
        ol.adam_step(ol.scalars(step=step, weight_decay=wd, adamw=adamw, grad_scale=0.5), *b, g,
                     pb)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x.view(np.uint32), y.view(np.uint32))
    np.testing.assert_array_equal(pa, pb)


@pytest.mark.parametrize("mode", ["adam", "adamw", "l2"])
@pytest.mark.parametrize("offset", [0, 3])
def test_host_adam_f32grad_bit_exact(mode, offset):
    """ptk_cpu_adam_f32grad (the offloaded chunk's update from a fp32
    reduce-scattered sum, the offload path's peer reduce-scatter): every rule,
    unaligned output, a NaN in the gradients, statistics -- bit-identical to
    the oracle's fp32-gradient step."""
    from paper_2406_08334_b200 import _native as nat
    n = 50_021
    wd, adamw = {"adam": (0.0, False), "adamw": (0.01, True), "l2": (0.01, False)}[mode]
    master = ol.fill_f32(n, 5, 0.05)
    g = ol.fill_f32(n, 6, 2e-3)
    g[11] = np.nan
    a = [master.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)]
    b = [master.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)]
    buf = np.zeros(n + 8, np.uint16)
    pa = buf[offset:offset + n]
    pb = np.zeros(n, np.uint16)
    for step in (1, 2):
        cfg = nat.adam_config(step=step, weight_decay=wd, adamw=adamw, grad_scale=0.25)
        sq, bad = ctypes.c_double(), ctypes.c_int64()
        nat.lib.ptk_cpu_adam_f32grad(ctypes.byref(cfg),
                                     *[ctypes.c_void_p(x.ctypes.data) for x in a],
                                     ctypes.c_void_p(g.ctypes.data),
                                     ctypes.c_void_p(pa.ctypes.data), n, 2, ctypes.byref(sq),
                                     ctypes.byref(bad))
        osq, obad = ol.adam_step(ol.scalars(step=step, weight_decay=wd, adamw=adamw,
                                            grad_scale=0.25), *b, g, pb)
        assert bad.value == obad == 1
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x.view(np.uint32), y.view(np.uint32))
    np.testing.assert_array_equal(pa, pb)


def test_peer_exchange_argument_errors_without_a_gpu():
    """The peer exchange and the symmetric-window entry points validate their
    arguments before touching the device: loud PTK_EINVAL with the entry
    point's name (runs on the CPU box)."""
    from paper_2406_08334_b200 import _native as nat
    arr = (ctypes.c_void_p * nat.PTK_MAX_PEERS)()
    out = ctypes.c_void_p(16)
    cases = [
        (lambda: nat.raw.ptk_peer_reduce_scatter_f32(None, 2, 0, 8, out, None),
         "ptk_peer_reduce_scatter_f32"),
        (lambda: nat.raw.ptk_peer_reduce_scatter_f32(arr, 9, 0, 8, out, None),
         "ptk_peer_reduce_scatter_f32"),
        (lambda: nat.raw.ptk_peer_reduce_scatter_f32(arr, 2, 2, 8, out, None),
         "ptk_peer_reduce_scatter_f32"),
        (lambda: nat.raw.ptk_peer_reduce_scatter_f32(arr, 2, 0, 8, out, None),   # null peers
         "null peer"),
        (lambda: nat.raw.ptk_peer_allgather(None, 2, 0, 16, None), "ptk_peer_allgather"),
        (lambda: nat.raw.ptk_peer_allgather(arr, 2, 0, -1, None), "ptk_peer_allgather"),
        (lambda: nat.raw.ptk_peer_allgather(arr, 2, 1, 16, None), "null local buffer"),
        (lambda: nat.raw.ptk_comm_window_register(None, out, 16, ctypes.byref(ctypes.c_void_p())),
         "null comm"),
        (lambda: nat.raw.ptk_comm_mem_alloc(None, 16), "ptk_comm_mem_alloc"),
        (lambda: nat.raw.ptk_cpu_adam_f32grad(None, None, None, None, None, None, 0, 0, None,
                                              None), "ptk_cpu_adam_f32grad"),
    ]
    for call, what in cases:
        assert call() == nat.PTK_EINVAL, what
        assert what in nat.last_error(), (what, nat.last_error())


def test_errors_are_reported():
    from paper_2406_08334_b200 import _native as nat
    rc = nat.raw.ptk_cpu_adam(None, None, None, None, None, None, 0, 0, None, None)
    assert rc == nat.PTK_OK - 1
    assert "ptk_cpu_adam" in nat.last_error()
    assert nat.shard_elems(-1, 1) == -1


def test_host_profile_probe_and_argument_checks():
    """ptk_profile_cpu_adam_rate is host-only (K6): it runs without a GPU."""
    from paper_2406_08334_b200 import _native as nat
    rate = ctypes.c_double()
    assert nat.raw.ptk_profile_cpu_adam_rate(1 << 20, ctypes.byref(rate)) == nat.PTK_OK
    assert rate.value > 1e6
    assert nat.raw.ptk_profile_cpu_adam_rate(0, ctypes.byref(rate)) != nat.PTK_OK
    assert "ptk_profile_cpu_adam_rate" in nat.last_error()
    assert nat.raw.ptk_profile_collective(None, 2, 1 << 20, None, None) != nat.PTK_OK


def test_planner_first_then_torch_in_a_fresh_process():
    """The first thing a process touches may be the planner (libptk.so) and
    only later torch: torch's NCCL must still be the one the process binds
    (a regression of the reference arm: `import torch` after libptk failed
    with `undefined symbol: ncclDevCommCreate`)."""
    import subprocess
    import sys
    code = ("from paper_2406_08334_b200 import planner\n"
            "planner.layout_for('gpt2-1b_b2')\n"
            "import torch, torch.distributed\n"
            "print(torch.zeros(2).sum().item())\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=REPO,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
