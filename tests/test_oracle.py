"""Pin the data-plane oracle (oracle/chunk_step.c) before trusting it.

The reference never executes optimizer numerics, so there are no
golden vectors for them in /root/reference; the oracle's Adam is pinned here
against torch 2.11's own torch.optim.Adam / AdamW (single-tensor path), and its
bf16 rounding / generator against numpy and torch.
"""
import numpy as np
import pytest
import torch

import oracle_lib as ol


def _torch_run(master, grads, steps, adamw, wd, lr=1e-3):
    p = torch.nn.Parameter(torch.from_numpy(master.copy()))
    cls = torch.optim.AdamW if adamw else torch.optim.Adam
    opt = cls([p], lr=lr, betas=(0.9, 0.999), eps=1e-8, weight_decay=wd, foreach=False,
              fused=False)
    for t in range(steps):
        p.grad = torch.from_numpy(ol.bf16_to_f32(grads[t]).copy())
        opt.step()
    st = opt.state[p]
    return p.detach().numpy(), st["exp_avg"].numpy(), st["exp_avg_sq"].numpy()


@pytest.mark.parametrize("adamw,wd", [(False, 0.0), (True, 0.01), (False, 0.01)])
def test_oracle_adam_matches_torch_10_steps(adamw, wd):
    n = 4099
    master = ol.fill_f32(n, 0, 0.05)
    grads = [ol.fill_bf16(n, 1 + t, 1e-3) for t in range(10)]
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    p = master.copy()
    for t in range(10):
        ol.adam_step(ol.scalars(weight_decay=wd, adamw=adamw, step=t + 1), p, m, v, grads[t])
    tp, tm, tv = _torch_run(master, grads, 10, adamw, wd)
    # fp32 master/m/v rel <= 1e-6 after 10 steps (IEEE div/sqrt).
    # torch's CPU lerp_/addcmul_ kernels may fuse (FMA); the oracle does not, so
    # elements whose EMA nearly cancels differ by a few ulps of the array
    # scale: the tolerance is relative to max|x| for m and v.
    np.testing.assert_allclose(p, tp, rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(m, tm, rtol=1e-6, atol=1e-6 * np.abs(tm).max())
    np.testing.assert_allclose(v, tv, rtol=1e-6, atol=1e-6 * np.abs(tv).max())


def test_bf16_rounding_matches_torch():
    x = np.concatenate([ol.fill_f32(100000, 7, 3.0),
                        np.array([0.0, -0.0, 1e-40, -1e-40, 3.4e38, np.inf, -np.inf],
                                 np.float32)])
    ours = np.array([ol.lib.oracle_f32_to_bf16(float(f)) for f in x[:2000]], np.uint16)
    ref = torch.from_numpy(x[:2000]).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    np.testing.assert_array_equal(ours, ref)
    np.testing.assert_array_equal(ol.f32_to_bf16(x), torch.from_numpy(x).to(torch.bfloat16)
                                  .view(torch.int16).numpy().view(np.uint16))
    assert ol.lib.oracle_f32_to_bf16(float("nan")) == 0x7FFF


def test_generator_is_counter_based():
    a = ol.fill_f32(1000, 5, 1.0)
    b = ol.fill_f32(300, 5, 1.0, index0=700)
    np.testing.assert_array_equal(a[700:], b)
    assert a.min() >= -1.0 and a.max() < 1.0
    # u = k * 2^-23 - 1 with k a 24-bit integer: exactly representable
    k = (a.astype(np.float64) + 1.0) * 2 ** 23
    np.testing.assert_array_equal(k, np.round(k))


def test_stats_sumsq_and_nonfinite():
    n = 1000
    g = ol.fill_bf16(n, 3, 1e-3)
    g[5] = 0x7F80   # +inf
    g[17] = 0xFFC0  # nan
    master = ol.fill_f32(n, 0, 0.05)
    m = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    sq, bad = ol.adam_step(ol.scalars(step=1, grad_scale=0.5), master, m, v, g)
    assert bad == 2


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_mapping_and_collectives(world):
    n = 1001
    shard = ol.shard_elems(n, world)
    assert shard % 8 == 0 and shard * world >= n and shard * world - n < 8 * world
    grads = [ol.fill_bf16(shard * world, 10 + r, 1.0) for r in range(world)]
    total = sum(ol.bf16_to_f32(g).astype(np.float64) for g in grads)
    for r in range(world):
        f = ol.reduce_scatter(grads, r, shard, fp32=True)
        np.testing.assert_allclose(f, total[r * shard:(r + 1) * shard], rtol=1e-6, atol=1e-6)
    shards = [np.arange(shard, dtype=np.uint16) + r for r in range(world)]
    full = ol.allgather(shards)
    np.testing.assert_array_equal(full, np.concatenate(shards))
