"""The seeded input generator: deterministic, shard-consistent, shaped like the
paper's workloads; its GPU twin is bit-identical to the numpy recipe."""
import numpy as np
import pytest

import synth


def test_deterministic_and_seeded():
    e = synth.col_scale_init(300, layer=3)
    a = synth.grad(17, 300, layer=3, step=5, scale_exp=e)
    b = synth.grad(17, 300, layer=3, step=5, scale_exp=e)
    c = synth.grad(17, 300, layer=3, step=6, scale_exp=e)
    assert a.dtype == np.uint16 and np.array_equal(a, b) and not np.array_equal(a, c)


def test_row_shards_concatenate():
    e = synth.col_scale_init(64, layer=1)
    whole = synth.grad(40, 64, 1, 2, e)
    parts = [synth.grad(10, 64, 1, 2, e, row0=10 * r) for r in range(4)]
    assert np.array_equal(np.concatenate(parts), whole)
    assert np.array_equal(np.concatenate([synth.param(20, 64, 1, row0=0), synth.param(20, 64, 1, row0=20)]),
                          synth.param(40, 64, 1))


def test_values_exact_in_fp32_and_column_structure():
    e = synth.col_scale_init(512, layer=0)
    g32 = synth.grad(256, 512, 0, 0, e, dtype="fp32")
    # an 18-bit integer times a power of two: the fp32 value is exact, |z| <= 2 * 2^(e-10)
    z = g32 / np.ldexp(1.0, e.astype(np.int32) - 26)[None, :]
    assert np.array_equal(z, np.round(z)) and np.all(np.abs(z) <= 131070)
    # column-concentrated energy (P:204 reports the top 1% of gradients carrying ~89% of norm^2)
    col = (g32.astype(np.float64) ** 2).sum(0)
    top = np.sort(col)[::-1]
    assert top[: len(top) // 10].sum() / top.sum() > 0.5


def test_scale_redraw_rate_calibrated():
    """~0.03% of the column scales are redrawn per step (P:328 calibration, synth module doc)."""
    m = 400000
    j = np.arange(m, dtype=np.uint64)
    hr = synth._hash(synth.stream_key(synth.SEED, synth.TAG_REDRAW, 2, 1), j)
    frac = np.mean((hr & np.uint64(0xFFFFFFFF)) < np.uint64(synth.REDRAW_THRESHOLD))
    assert 0.00022 < frac < 0.00038
    e0 = synth.col_scale_init(m, layer=2)
    e1 = synth.col_scale_advance(e0, 1, layer=2)
    assert np.mean(e0 != e1) <= frac


def test_top1pct_retention_by_fixed_top10pct_channels():
    """P:328 (fig. ratention_rate): the top-10% channels chosen at step 0 keep > 95% of each
    later step's top-1% elements across 100 steps.  Checked on a 512 x 4096 matrix at
    steps 1, 50 and 99 (element top-1% by magnitude; channels by column L2 norm)."""
    from synth import host
    n, m = 512, 4096
    e0 = host.col_scale_at(m, 0, 0)
    G0 = host.grad(n, m, 0, 0, e0, "fp32").astype(np.float64)
    sel = np.argsort(-(G0 ** 2).sum(0), kind="stable")[: m // 10]
    mask = np.zeros(m, bool)
    mask[sel] = True
    for t in (1, 50, 99):
        G = np.abs(host.grad(n, m, 0, t, host.col_scale_at(m, t, 0), "fp32"))
        kth = np.partition(G.ravel(), -(n * m // 100))[-(n * m // 100)]
        top = G >= kth
        assert top[:, mask].sum() / top.sum() > 0.95, t


def test_tie_mode_has_ties():
    g = synth.grad_tie(8, 100, 0, 0, dtype="fp32")
    assert set(np.unique(g * 256).tolist()) <= {-2.0, -1.0, 0.0, 1.0, 2.0}


def test_model_shapes():
    L7 = synth.llama2_7b_linears()
    assert len(L7) == 225 and sum(n * m for _, n, m in L7) == 6_607_077_376
    L13 = synth.llama2_13b_linears()
    assert len(L13) == 281 and sum(n * m for _, n, m in L13) == 12_851_609_600
    G2 = synth.gpt2_small_linears()
    assert len(G2) == 49 and sum(n * m for _, n, m in G2) == 123_532_032


@pytest.mark.gpu
def test_gpu_generator_bit_identical():
    import torch
    from synth import gpu
    for dt, tdt in (("bf16", torch.bfloat16), ("fp32", torch.float32)):
        n, m, layer = 333, 1000, 7
        sc = gpu.ColScale(m, layer)
        sc.advance_to(3)
        out = torch.empty(n, m, dtype=tdt, device="cuda")
        gpu.fill_grad(out, layer, 3, sc, row0=50)
        e = synth.col_scale_at(m, 3, layer)
        assert np.array_equal(sc.e.cpu().numpy(), e)
        want = synth.grad(n, m, layer, 3, e, dtype=dt, row0=50)
        got = out.cpu().view(torch.int16).numpy().view(np.uint16) if dt == "bf16" else out.cpu().numpy()
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), dt
        gpu.fill_param(out, layer, row0=50)
        want = synth.param(n, m, layer, dtype=dt, row0=50)
        got = out.cpu().view(torch.int16).numpy().view(np.uint16) if dt == "bf16" else out.cpu().numpy()
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), dt
        gpu.fill_grad_tie(out, layer, 2)
        want = synth.grad_tie(n, m, layer, 2, dtype=dt)
        got = out.cpu().view(torch.int16).numpy().view(np.uint16) if dt == "bf16" else out.cpu().numpy()
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), dt


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_host_c_twin_bit_identical(dtype):
    """synth/synth_host.c (used to generate full-size inputs for the CPU-oracle timing) is
    bit-identical to the numpy recipe: scales over several steps, gradients, params, shards."""
    from synth import host
    for m, layer, step in ((300, 3, 0), (4096, 7, 5), (257, 1, 12)):
        e = synth.col_scale_at(m, step, layer)
        assert np.array_equal(host.col_scale_at(m, step, layer), e)
        assert np.array_equal(host.grad(9, m, layer, step, e, dtype, row0=13),
                              synth.grad(9, m, layer, step, e, dtype, row0=13))
        assert np.array_equal(host.param(5, m, layer, dtype, row0=2), synth.param(5, m, layer, dtype, row0=2))
