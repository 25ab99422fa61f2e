"""GPU parity of the fused chunk Adam (K1+K2) through the C-ABI.

Checked BIT-EXACTLY against oracle/chunk_step.c (same update rule, same fp32
scalars, no FMA contraction on either side): master, exp_avg, exp_avg_sq and
the bf16 parameter copy. Gradient statistics: non-finite count exact, sum of
squares within 1e-6 relative (fp32 per-thread / fp64 cross-CTA accumulation vs
the oracle's fp64 per element).
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle_lib as ol

pytestmark = pytest.mark.gpu


def _nat():
    from paper_2406_08334_b200 import _native
    return _native


def _vp(t):
    return ctypes.c_void_p(t.data_ptr())


def _dev_f32(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _dev_bits16(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(dev)


def _bits(t):
    x = t.cpu().numpy()
    return x.view(np.uint32) if x.dtype == np.float32 else x.view(np.uint16)


class DevState:
    def __init__(self, master, dev, grad_f32=False):
        n = master.size
        self.n = n
        self.master = _dev_f32(master, dev)
        self.m = torch.zeros(n, dtype=torch.float32, device=dev)
        self.v = torch.zeros(n, dtype=torch.float32, device=dev)
        self.p = torch.zeros(max(n, 1), dtype=torch.int16, device=dev)
        nat = _nat()
        self.ws = torch.zeros(int(nat.raw.ptk_stats_workspace_bytes()), dtype=torch.uint8,
                              device=dev)
        self.stats = torch.zeros(2, dtype=torch.float64, device=dev)

    def step(self, cfg, grad_dev, f32=False, gscale_dev=None, skip_dev=None, stats=True):
        nat = _nat()
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        fn = nat.lib.ptk_chunk_adam_f32grad if f32 else nat.lib.ptk_chunk_adam
        nat.lib.ptk_stats_reset(_vp(self.stats), s)
        fn(ctypes.byref(cfg), _vp(self.master), _vp(self.m), _vp(self.v), _vp(grad_dev),
           _vp(self.p), self.n, _vp(self.stats) if stats else None,
           _vp(self.ws), _vp(gscale_dev) if gscale_dev is not None else None,
           _vp(skip_dev) if skip_dev is not None else None, s)


@pytest.mark.parametrize("n", [1, 7, 8, 9, 255, 1536, 4096, 1536 * 148, 1536 * 148 * 3 + 8,
                               1_000_003, (1 << 22) + 5])
@pytest.mark.parametrize("mode", ["adam", "adamw", "l2"])
def test_chunk_adam_bit_exact(cuda_device, n, mode):
    nat = _nat()
    adamw = mode == "adamw"
    wd = 0.0 if mode == "adam" else 0.01
    master = ol.fill_f32(n, 0, 0.05)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    out = np.zeros(n, np.uint16)
    st = DevState(master, cuda_device)
    for step in range(1, 4):
        g = ol.fill_bf16(n, 100 + step, 1e-3)
        gscale = 0.5 if step == 2 else 1.0
        cfg = nat.adam_config(lr=1e-3, weight_decay=wd, adamw=adamw, step=step, grad_scale=gscale)
        st.step(cfg, _dev_bits16(g, cuda_device))
        sq, bad = ol.adam_step(ol.scalars(weight_decay=wd, adamw=adamw, step=step,
                                          grad_scale=gscale), master, m, v, g, out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(st.master), master.view(np.uint32))
    np.testing.assert_array_equal(_bits(st.m), m.view(np.uint32))
    np.testing.assert_array_equal(_bits(st.v), v.view(np.uint32))
    np.testing.assert_array_equal(_bits(st.p)[:n], out)
    dsq = float(st.stats[0])
    dbad = int(st.stats.view(torch.int64)[1])
    assert dbad == bad == 0
    assert abs(dsq - sq) <= 1e-6 * sq + 1e-30


def test_chunk_adam_f32grad_bit_exact(cuda_device):
    nat = _nat()
    n = 300_017
    master = ol.fill_f32(n, 1, 0.05)
    g = ol.fill_f32(n, 2, 2e-3)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    out = np.zeros(n, np.uint16)
    st = DevState(master, cuda_device)
    cfg = nat.adam_config(step=1, grad_scale=0.25)
    st.step(cfg, _dev_f32(g, cuda_device), f32=True)
    ol.adam_step(ol.scalars(step=1, grad_scale=0.25), master, m, v, g, out)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(st.master), master.view(np.uint32))
    np.testing.assert_array_equal(_bits(st.p)[:n], out)


def test_nonfinite_counted_and_skip_flag(cuda_device):
    nat = _nat()
    n = 10_000
    master = ol.fill_f32(n, 0, 0.05)
    g = ol.fill_bf16(n, 3, 1e-3)
    g[[5, 77, 9999]] = [0x7F80, 0xFF80, 0x7FC0]  # +inf, -inf, nan
    st = DevState(master, cuda_device)
    st.step(nat.adam_config(step=1), _dev_bits16(g, cuda_device))
    torch.cuda.synchronize()
    assert int(st.stats.view(torch.int64)[1]) == 3
    # skip flag set -> the launch is a no-op
    before = _bits(st.master).copy()
    skip = torch.ones(1, dtype=torch.int32, device=cuda_device)
    st.step(nat.adam_config(step=2), _dev_bits16(g, cuda_device), skip_dev=skip)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(st.master), before)


def test_grad_stats_and_clip_coef(cuda_device):
    nat = _nat()
    n = 1_234_567
    g = ol.fill_bf16(n, 9, 1e-2)
    gd = _dev_bits16(g, cuda_device)
    out = torch.zeros(n, dtype=torch.float32, device=cuda_device)
    ws = torch.zeros(int(nat.raw.ptk_stats_workspace_bytes()), dtype=torch.uint8,
                     device=cuda_device)
    stats = torch.zeros(2, dtype=torch.float64, device=cuda_device)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.lib.ptk_stats_reset(_vp(stats), s)
    nat.lib.ptk_grad_stats(_vp(gd), n, 0.5, _vp(out), _vp(stats), _vp(ws), s)
    coef = torch.zeros(1, dtype=torch.float32, device=cuda_device)
    skip = torch.full((1,), 7, dtype=torch.int32, device=cuda_device)
    nat.lib.ptk_clip_coef(_vp(stats), 1.0, _vp(coef), _vp(skip), s)
    torch.cuda.synchronize()
    ref = ol.bf16_to_f32(g) * np.float32(0.5)
    np.testing.assert_array_equal(out.cpu().numpy(), ref)
    sq = float(np.sum(ref.astype(np.float64) ** 2))
    assert abs(float(stats[0]) - sq) <= 1e-6 * sq
    norm = np.sqrt(sq)
    assert abs(float(coef[0]) - min(1.0, 1.0 / (norm + 1e-6))) <= 1e-6
    assert int(skip[0]) == 0
    # ptk_grad_prep (SURVEY §8(b) K2 name) = the cast/scale with a required output
    out2 = torch.zeros_like(out)
    stats2 = torch.zeros_like(stats)
    assert nat.raw.ptk_grad_prep(_vp(gd), n, 0.5, None, _vp(stats2), _vp(ws), s) != nat.PTK_OK
    nat.lib.ptk_grad_prep(_vp(gd), n, 0.5, _vp(out2), _vp(stats2), _vp(ws), s)
    torch.cuda.synchronize()
    assert torch.equal(out2, out) and torch.equal(stats2, stats)


def test_gscale_dev_multiplies(cuda_device):
    nat = _nat()
    n = 4096
    master = ol.fill_f32(n, 0, 0.05)
    g = ol.fill_bf16(n, 3, 1e-3)
    a = DevState(master, cuda_device)
    b = DevState(master, cuda_device)
    two = torch.full((1,), 2.0, dtype=torch.float32, device=cuda_device)
    a.step(nat.adam_config(step=1, grad_scale=0.5), _dev_bits16(g, cuda_device), gscale_dev=two)
    b.step(nat.adam_config(step=1, grad_scale=1.0), _dev_bits16(g, cuda_device))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(a.master), _bits(b.master))


def test_invalid_arguments_fail_loudly(cuda_device):
    nat = _nat()
    n = 64
    st = DevState(ol.fill_f32(n, 0, 0.05), cuda_device)
    g = torch.zeros(n + 8, dtype=torch.int16, device=cuda_device)
    misaligned = ctypes.c_void_p(g.data_ptr() + 2)
    cfg = nat.adam_config(step=1)
    rc = nat.raw.ptk_chunk_adam(ctypes.byref(cfg), _vp(st.master), _vp(st.m), _vp(st.v),
                                misaligned, None, n, None, None, None, None, None)
    assert rc == -1 and "aligned" in nat.last_error()
    bad = nat.adam_config(step=0)
    rc = nat.raw.ptk_chunk_adam(ctypes.byref(bad), _vp(st.master), _vp(st.m), _vp(st.v),
                                _vp(g), None, n, None, None, None, None, None)
    assert rc == -1
    with pytest.raises(nat.PtkError):
        nat.lib.ptk_chunk_adam(ctypes.byref(bad), _vp(st.master), _vp(st.m), _vp(st.v),
                               _vp(g), None, n, None, None, None, None, None)


def test_fill_matches_oracle(cuda_device):
    nat = _nat()
    n = 100_003
    a = torch.empty(n, dtype=torch.float32, device=cuda_device)
    b = torch.empty(n, dtype=torch.int16, device=cuda_device)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.lib.ptk_fill_uniform_f32(_vp(a), n, 42, 1000, 0.05, s)
    nat.lib.ptk_fill_uniform_bf16(_vp(b), n, 43, 7, 1e-3, s)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(a), ol.fill_f32(n, 42, 0.05, 1000).view(np.uint32))
    np.testing.assert_array_equal(_bits(b), ol.fill_bf16(n, 43, 1e-3, 7))


# ---- one launch over a chunk table (ptk_chunk_adam_table) ----

TABLE_CASES = {
    # unpadded lengths (n % 8 tails), empty and sub-tile chunks, many small chunks
    "ragged": [1, 7, 0, 8, 1536, 1536 * 148 + 8, 100_003, 5, 4096, 0, 1537],
    "many_small": [12_288 + 8 * i for i in range(64)],
    "one_big": [1536 * 148 * 5 + 24],
    # more chunks than one launch's table capacity (launched in batches)
    "over_capacity": [2048 * (1 + i % 5) + 8 * (i % 3) + (i % 7) for i in range(300)],
}


def _random_table(seed: int) -> list[int]:
    """Seeded random tables: empty, sub-unit, tile-boundary (+-1) and
    multi-tile chunks, 1..200 of them."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(int(rng.integers(1, 201))):
        kind = rng.integers(0, 4)
        if kind == 0:
            out.append(int(rng.integers(0, 9)))
        elif kind == 1:
            out.append(int(rng.integers(9, 5000)))
        elif kind == 2:
            out.append(int(2048 * rng.integers(1, 40) + rng.integers(-1, 2)))
        else:
            out.append(int(rng.integers(5000, 400_000)))
    return out


for _seed in range(6):
    TABLE_CASES[f"random{_seed}"] = _random_table(_seed)


@pytest.mark.parametrize("case", sorted(TABLE_CASES))
def test_chunk_table_bit_exact(cuda_device, case):
    """Every chunk of a table updated by ONE persistent TMA launch (tiles of
    all chunks walked by each CTA in global order): bit-identical to the
    oracle per chunk, statistics summed over the whole table."""
    nat = _nat()
    sizes = TABLE_CASES[case]
    states, host = [], []
    for i, n in enumerate(sizes):
        master = ol.fill_f32(n, 500 + i, 0.05)
        states.append(DevState(master, cuda_device))
        host.append([master, np.zeros(n, np.float32), np.zeros(n, np.float32),
                     np.zeros(n, np.uint16)])
    grads = [_dev_bits16(ol.fill_bf16(n, 900 + i, 1e-3), cuda_device) for i, n in enumerate(sizes)]
    descs = (nat.ChunkDesc * len(sizes))()
    for d, st, g in zip(descs, states, grads):
        d.master, d.exp_avg, d.exp_avg_sq = st.master.data_ptr(), st.m.data_ptr(), st.v.data_ptr()
        d.grad, d.param_out, d.n = g.data_ptr(), st.p.data_ptr(), st.n
    table = ctypes.c_void_p()
    nat.lib.ptk_chunk_table_create(descs, len(sizes), ctypes.byref(table))
    assert nat.raw.ptk_chunk_table_params(table) == sum(sizes)
    ws, stats = states[0].ws, states[0].stats
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    want_sq = 0.0
    for step in (1, 2, 3):
        cfg = nat.adam_config(lr=1e-3, weight_decay=0.01, adamw=True, step=step,
                              grad_scale=0.5 if step == 2 else 1.0)
        nat.lib.ptk_stats_reset(_vp(stats), s)
        nat.lib.ptk_chunk_adam_table(ctypes.byref(cfg), table, _vp(stats), _vp(ws), None, None, s)
        want_sq = 0.0
        for i, (n, h) in enumerate(zip(sizes, host)):
            sq, _ = ol.adam_step(ol.scalars(lr=1e-3, weight_decay=0.01, adamw=True, step=step,
                                            grad_scale=0.5 if step == 2 else 1.0),
                                 h[0], h[1], h[2], ol.fill_bf16(n, 900 + i, 1e-3), h[3])
            want_sq += sq
    torch.cuda.synchronize()
    for st, h, n in zip(states, host, sizes):
        np.testing.assert_array_equal(_bits(st.master), h[0].view(np.uint32))
        np.testing.assert_array_equal(_bits(st.m), h[1].view(np.uint32))
        np.testing.assert_array_equal(_bits(st.v), h[2].view(np.uint32))
        np.testing.assert_array_equal(_bits(st.p)[:n], h[3])
    assert abs(float(stats[0]) - want_sq) <= 1e-6 * want_sq
    # device skip flag: the whole table is a no-op
    before = [_bits(st.master).copy() for st in states]
    skip = torch.ones(1, dtype=torch.int32, device=cuda_device)
    cfg = nat.adam_config(step=4)
    nat.lib.ptk_chunk_adam_table(ctypes.byref(cfg), table, None, None, None, _vp(skip), s)
    torch.cuda.synchronize()
    for b, st in zip(before, states):
        np.testing.assert_array_equal(_bits(st.master), b)
    nat.lib.ptk_chunk_table_destroy(table)


def test_chunk_table_graph_capture_and_bad_args(cuda_device):
    nat = _nat()
    n = 50_000
    st = DevState(ol.fill_f32(n, 1, 0.05), cuda_device)
    ref = DevState(ol.fill_f32(n, 1, 0.05), cuda_device)
    g = _dev_bits16(ol.fill_bf16(n, 2, 1e-3), cuda_device)
    d = (nat.ChunkDesc * 1)()
    d[0].master, d[0].exp_avg, d[0].exp_avg_sq = st.master.data_ptr(), st.m.data_ptr(), st.v.data_ptr()
    d[0].grad, d[0].param_out, d[0].n = g.data_ptr(), st.p.data_ptr(), n
    table = ctypes.c_void_p()
    nat.lib.ptk_chunk_table_create(d, 1, ctypes.byref(table))
    graph = torch.cuda.CUDAGraph()
    cfgs = [nat.adam_config(step=k) for k in (1, 2)]
    with torch.cuda.graph(graph):
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        for cfg in cfgs:
            nat.lib.ptk_chunk_adam_table(ctypes.byref(cfg), table, None, None, None, None, s)
    graph.replay()
    for cfg in cfgs:
        ref.step(cfg, g, stats=False)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(_bits(st.master), _bits(ref.master))
    np.testing.assert_array_equal(_bits(st.p), _bits(ref.p))
    nat.lib.ptk_chunk_table_destroy(table)
    # misaligned buffers are refused at creation
    d[0].grad = g.data_ptr() + 2
    t2 = ctypes.c_void_p()
    assert nat.raw.ptk_chunk_table_create(d, 1, ctypes.byref(t2)) == -1
    assert "aligned" in nat.last_error()
