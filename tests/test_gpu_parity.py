"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by
element, on the same seeded inputs.  Bars (BASELINE.json north_star): selection
and compaction bit-exact (boundary swaps allowed only within the norm tolerance,
reading R3), norms within rel 1e-5, fp32 params/moments within rel 1e-6 and bf16
params within 1 ulp -- the kernels follow the oracle's op order, so the update
is also checked bit for bit."""
import math
import os

import numpy as np
import pytest
import torch

import synth
from gpu_util import (assert_bits_equal, assert_close_rel, bf16_ulp_diff, from_np, selection_ok, to_np)

pytestmark = pytest.mark.gpu

TDT = {"bf16": torch.bfloat16, "fp32": torch.float32}


@pytest.fixture(scope="module")
def zf():
    from paper_2505_12242_b200 import _build
    _build.build()
    from paper_2505_12242_b200 import zf as z
    return z


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle as o
    o.lib()
    return o


@pytest.fixture(scope="module")
def gpu():
    from synth import gpu as g
    return g


def _grad(gpu, n, m, dt, layer=0, step=0, ld=None, tie=False):
    ld = ld or m
    buf = torch.empty(n, ld, dtype=TDT[dt], device="cuda")
    G = buf[:, :m]
    if tie:
        gpu.fill_grad_tie(G, layer, step)
    else:
        sc = gpu.ColScale(m, layer)
        sc.advance_to(step)
        gpu.fill_grad(G, layer, step, sc)
    return G


# ------------------------------------------------------------------ K1 norms
NORM_CASES = [(256, 512, "fp32", None), (4096, 4096, "bf16", None), (1000, 1000, "bf16", None),
              (37, 1001, "bf16", 1003), (130, 257, "fp32", None), (513, 768, "bf16", 776), (1, 9, "bf16", None),
              (11008, 4096, "bf16", None), (300, 13824, "bf16", None)]


@pytest.mark.parametrize("n,m,dt,ld", NORM_CASES)
def test_column_norms(zf, orc, gpu, n, m, dt, ld):
    G = _grad(gpu, n, m, dt, layer=n % 7, ld=ld)
    out = torch.full((m,), -1.0, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    zf.zf_column_norms(G, out, flag)
    out2 = torch.empty_like(out)
    zf.zf_column_norms(G, out2)
    torch.cuda.synchronize()
    want = orc.column_norms(np.ascontiguousarray(to_np(G)))
    got = to_np(out)
    assert_close_rel(got, want, 1e-5, "norms")
    assert_bits_equal(to_np(out2), got, "norms determinism")
    assert int(flag.item()) == 0


def test_column_norms_tie_heavy_exact(zf, orc, gpu):
    # tie-heavy values are multiples of 2^-8 with small sums: every partial sum is exact
    G = _grad(gpu, 200, 3000, "bf16", tie=True)
    out = torch.empty(3000, device="cuda")
    zf.zf_column_norms(G, out)
    assert_bits_equal(to_np(out), orc.column_norms(to_np(G)), "tie norms")


def test_column_norms_nonfinite_flag(zf, gpu):
    G = _grad(gpu, 300, 512, "bf16")
    G[123, 77] = float("nan")
    out = torch.empty(512, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    zf.zf_column_norms(G, out, flag)
    assert int(flag.item()) == 1


# ------------------------------------------------------------------ K2 top-k
@pytest.mark.parametrize("m,ppm", [(8, 250000), (100, 100000), (768, 100000), (768, 10000), (4096, 100000),
                                   (4096, 10000), (11008, 100000), (13824, 10000), (50000, 100000), (5000, 1),
                                   (333, 1000000)])
def test_topk_exact(zf, orc, m, ppm):
    rng = np.random.default_rng(m + ppm)
    norms = (rng.standard_normal(m) ** 2 * np.exp(rng.standard_normal(m) * 2)).astype(np.float32)
    norms[rng.choice(m, m // 5, replace=False)] = norms[0]          # many exact ties incl. at the boundary
    k = orc.k_for(m, ppm)
    idx = torch.empty(k, dtype=torch.int32, device="cuda")
    zf.zf_topk_columns(from_np(norms), k, idx)
    assert to_np(idx).tolist() == orc.topk(norms, k).tolist()


def test_topk_integer_ties(zf, orc):
    rng = np.random.default_rng(5)
    for m in (1, 2, 31, 32, 33, 1000, 4097):
        norms = rng.integers(0, 4, m).astype(np.float32)
        for k in sorted({1, max(1, m // 3), m}):
            idx = torch.empty(k, dtype=torch.int32, device="cuda")
            zf.zf_topk_columns(from_np(norms), k, idx)
            assert to_np(idx).tolist() == orc.topk(norms, k).tolist(), (m, k)


# ------------------------------------------------------------------ K3 AdamW (standalone)
@pytest.mark.parametrize("n,m,gdt,pdt,wd,dec,ldp", [(256, 512, "fp32", "fp32", 0.0, 1, None),
                                                   (300, 4096, "bf16", "bf16", 0.0, 1, None),
                                                   (77, 1001, "bf16", "bf16", 0.01, 1, 1009),
                                                   (64, 640, "bf16", "fp32", 0.01, 0, None),
                                                   (50, 200, "fp32", "bf16", 0.01, 1, None)])
def test_selective_adam_bitexact(zf, orc, gpu, n, m, gdt, pdt, wd, dec, ldp):
    rng = np.random.default_rng(n * m)
    G = _grad(gpu, n, m, gdt, layer=1)
    Pbuf = torch.empty(n, ldp or m, dtype=TDT[pdt], device="cuda")
    P = Pbuf[:, :m]
    gpu.fill_param(P, 1)
    k = orc.k_for(m, 100000)
    idx_np = np.sort(rng.choice(m, k, replace=False)).astype(np.int32)
    M0 = (rng.standard_normal((n, k)) * 1e-3).astype(np.float32)
    V0 = (rng.random((n, k)) * 1e-6).astype(np.float32)
    st0 = rng.integers(0, 20, k).astype(np.int32)
    hp = orc.AdamHP(lr=1e-3, weight_decay=wd, decoupled=dec)
    Pn, Gn = np.ascontiguousarray(to_np(P)), np.ascontiguousarray(to_np(G))
    M1, V1, st1 = M0.copy(), V0.copy(), st0.copy()
    orc.selective_adamw(Pn, Gn, idx_np, M1, V1, st1, hp)
    Md, Vd, sd = from_np(M0), from_np(V0), from_np(st0)
    zf.zf_selective_adam(P, G, from_np(idx_np), Md, Vd, sd, zf.adam_params(lr=1e-3, weight_decay=wd, decoupled=dec))
    torch.cuda.synchronize()
    assert_bits_equal(to_np(sd), st1, "steps")
    assert_bits_equal(to_np(Md), M1, "exp_avg")
    assert_bits_equal(to_np(Vd), V1, "exp_avg_sq")
    assert_bits_equal(np.ascontiguousarray(to_np(P)), Pn, "params")
    if ldp:  # padding columns untouched
        pad = to_np(Pbuf[:, m:])
        assert np.array_equal(pad, to_np(Pbuf[:, m:]))


def _table_end(f):
    """First t >= 1 at which the fp32 bias-correction term f(t) (computed in double, rounded
    once) reaches its limit -- where the library's tables stop (the limit is used beyond)."""
    lim = np.float32(f(10 ** 9))
    t = 1
    while np.float32(f(t)) != lim:
        t += 1
    return t


def _ends(lr, b1, b2):
    return (_table_end(lambda t: lr / (1.0 - b1 ** t)), _table_end(lambda t: math.sqrt(1.0 - b2 ** t)))


@pytest.mark.parametrize("pdt", ["bf16", "fp32"])
def test_selective_adam_step_counts_past_the_tables(zf, orc, gpu, pdt):
    """Stateless AdamW at step counts straddling the ends of the bias-correction tables
    (ss = lr/(1-b1^t) reaches f32(lr) at t ~ 160, bc2s = sqrt(1-b2^t) reaches 1.0 at
    t ~ 1.7k for b2 = 0.99) and far beyond (2^20, 2^30): bit-exact vs the oracle, which
    evaluates both terms in double at every t (O6)."""
    n, m, lr, b1, b2 = 8, 4096, 1e-3, 0.9, 0.99
    e1, e2 = _ends(lr, b1, b2)
    cand = [0, 1, 2, e1 - 2, e1 - 1, e1, e1 + 1, e2 - 3, e2 - 2, e2 - 1, e2, e2 + 1, 5 * e2, 1 << 20, 1 << 30]
    k = len(cand) * 8
    rng = np.random.default_rng(17)
    st0 = np.array([cand[i % len(cand)] for i in range(k)], np.int32)
    idx_np = np.sort(rng.choice(m, k, replace=False)).astype(np.int32)
    G = _grad(gpu, n, m, "bf16", layer=3)
    P = torch.empty(n, m, dtype=TDT[pdt], device="cuda")
    gpu.fill_param(P, 3)
    M0 = (rng.standard_normal((n, k)) * 1e-3).astype(np.float32)
    V0 = (rng.random((n, k)) * 1e-6).astype(np.float32)
    hp = orc.AdamHP(lr=lr, beta1=b1, beta2=b2)
    Pn, Gn = np.ascontiguousarray(to_np(P)), np.ascontiguousarray(to_np(G))
    M1, V1, st1 = M0.copy(), V0.copy(), st0.copy()
    orc.selective_adamw(Pn, Gn, idx_np, M1, V1, st1, hp)
    Md, Vd, sd = from_np(M0), from_np(V0), from_np(st0)
    zf.zf_selective_adam(P, G, from_np(idx_np), Md, Vd, sd, zf.adam_params(lr=lr, beta1=b1, beta2=b2))
    torch.cuda.synchronize()
    assert_bits_equal(to_np(sd), st1, "steps")
    assert_bits_equal(to_np(Md), M1, "exp_avg")
    assert_bits_equal(to_np(Vd), V1, "exp_avg_sq")
    assert_bits_equal(np.ascontiguousarray(to_np(P)), Pn, "params")


def test_step_runs_past_the_bias_correction_tables(zf, orc, gpu):
    """zf_step (K3 with its per-slot {ss, bc2s} prologue) for more steps than the longer
    bias-correction table holds (b2 = 0.99: ~1.7k), one refresh at t = 0 and a fixed
    selection after it: parameters, moments and step counts bit-exact with the oracle at
    checkpoints on both sides of the table ends."""
    n, m, lr, b1, b2 = 16, 256, 1e-3, 0.9, 0.99
    e1, e2 = _ends(lr, b1, b2)
    T = e2 + 24
    N = 1 << 20
    ctx = zf.Context([zf.LayerShape(n, m)], topk_ratio_ppm=100000, refresh_interval=N, accum_interval=N,
                     adam=zf.adam_params(lr=lr, beta1=b1, beta2=b2))
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=N, accum_interval=N,
                        hp=orc.AdamHP(lr=lr, beta1=b1, beta2=b2))
    Gs = [_grad(gpu, n, m, "bf16", layer=5, step=j) for j in range(7)]     # cycled
    Gn = [np.ascontiguousarray(to_np(g)) for g in Gs]
    P = torch.empty(n, m, dtype=torch.bfloat16, device="cuda")
    gpu.fill_param(P, 5)
    Po = np.ascontiguousarray(to_np(P))
    checks = {e1 - 1, e1 + 1, e2 - 2, e2, e2 + 1, T - 1}
    for t in range(T):
        ctx.step(t, [Gs[t % 7]], [P])
        L.step(t, Gn[t % 7], Po)
        if t in checks:
            torch.cuda.synchronize()
            Md, Vd, sd = ctx.optimizer_state(0)
            assert np.array_equal(to_np(ctx.selected(0)), L.idx), t
            assert_bits_equal(to_np(sd), L.steps, f"steps t={t}")
            assert_bits_equal(to_np(Md), L.M, f"exp_avg t={t}")
            assert_bits_equal(to_np(Vd), L.V, f"exp_avg_sq t={t}")
            assert_bits_equal(np.ascontiguousarray(to_np(P)), Po, f"params t={t}")
    assert int(L.steps.max()) == T > e2
    ctx.close()


# ------------------------------------------------------------------ K3 compaction (standalone)
@pytest.mark.parametrize("n,m,dt,ld,ppm", [(256, 512, "fp32", None, 100000), (4096, 4096, "bf16", None, 100000),
                                           (1000, 1000, "bf16", None, 10000), (37, 1001, "bf16", 1003, 100000),
                                           (5, 20000, "bf16", None, 100000), (3, 40000, "fp32", None, 10000),
                                           (21, 768, "bf16", 776, 100000), (7, 13, "fp32", None, 500000),
                                           (9, 64, "bf16", None, 1000000)])
def test_compact_bitexact(zf, orc, gpu, n, m, dt, ld, ppm):
    rng = np.random.default_rng(n + m)
    G = _grad(gpu, n, m, dt, layer=2, ld=ld)
    k = orc.k_for(m, ppm)
    idx_np = np.sort(rng.choice(m, k, replace=False)).astype(np.int32)
    out = torch.full((max(1, n * (m - k)),), 7, dtype=TDT[dt], device="cuda")
    zf.zf_compact_unselected(G, from_np(idx_np), out)
    want = orc.compact(np.ascontiguousarray(to_np(G)), idx_np)
    assert_bits_equal(to_np(out)[: n * (m - k)].reshape(n, m - k), want, "compact")


@pytest.mark.parametrize("n,m,dt", [(512, 4096, "bf16"), (33, 1000, "fp32")])
def test_compact_into_pinned_host(zf, orc, gpu, n, m, dt):
    """Row 6/7 through the stateless primitive: K3 writes the compact block straight into
    pinned host memory (zero-copy over the host link, include/zf.h)."""
    rng = np.random.default_rng(n)
    G = _grad(gpu, n, m, dt, layer=4)
    k = orc.k_for(m, 100000)
    idx_np = np.sort(rng.choice(m, k, replace=False)).astype(np.int32)
    out = torch.full((n * (m - k),), 3, dtype=TDT[dt]).pin_memory()
    zf.zf_compact_unselected(G, from_np(idx_np), out)
    torch.cuda.synchronize()
    want = orc.compact(np.ascontiguousarray(to_np(G)), idx_np)
    assert_bits_equal(to_np(out).reshape(n, m - k), want, "compact (pinned host)")


# ------------------------------------------------------------------ zf_step vs oracle, multi-step
def _run_stateful(zf, orc, gpu, shapes, gdt, pdt, ppm, N, S, steps, offload, lr=1e-3, wd=0.0, check_every=1,
                  tie=False, ld_pad=0, cpu_update=False, warmup=0, state_offload=False, devacc=False,
                  cpu_async=False, side_stream=False, psub=True, poke=None, lagged=False, host_stages=0,
                  refresh_group_mb=0):
    hp_o = orc.AdamHP(lr=lr, weight_decay=wd)
    ctx = zf.Context([zf.LayerShape(n, m, m + ld_pad, m + ld_pad) for n, m in shapes], grad_dtype=TDT[gdt],
                     param_dtype=TDT[pdt], topk_ratio_ppm=ppm, refresh_interval=N, accum_interval=S,
                     adam=zf.adam_params(lr=lr, weight_decay=wd), offload=offload, host_accumulate=offload, cpu_update=cpu_update,
                     warmup_steps=warmup, state_offload=state_offload, device_accumulate=devacc,
                     cpu_update_async=cpu_async, param_subset=psub, lagged_selection=lagged,
                     host_stages=host_stages, refresh_group_mb=refresh_group_mb)
    scales = [gpu.ColScale(m, li) for li, (n, m) in enumerate(shapes)]
    Gs = [torch.empty(n, m + ld_pad, dtype=TDT[gdt], device="cuda")[:, :m] for n, m in shapes]
    Ps = [torch.empty(n, m + ld_pad, dtype=TDT[pdt], device="cuda")[:, :m] for n, m in shapes]
    for li, P in enumerate(Ps):
        gpu.fill_param(P, li)
    layers = [orc.OracleLayer(n=n, m=m, ratio_ppm=ppm, refresh_interval=N, accum_interval=S, hp=hp_o,
                              cpu_update=cpu_update, warmup=warmup, lagged=lagged) for n, m in shapes]
    Po = [np.ascontiguousarray(to_np(P)) for P in Ps]
    swaps = 0
    prevG = None
    for t in range(steps):
        for li, (G, sc) in enumerate(zip(Gs, scales)):
            if tie:
                gpu.fill_grad_tie(G, li, t)
            else:
                sc.advance_to(t)
                gpu.fill_grad(G, li, t, sc)
        Gn = [np.ascontiguousarray(to_np(G)) for G in Gs]
        if poke is not None and t in poke:
            # the caller writes the parameters outside zf_step (e.g. a checkpoint load): every
            # 3rd element of every parameter is negated, on the GPU and in the oracle's copy
            for li, P in enumerate(Ps):
                Pc = P.clone()
                Pc.view(-1)[::3] = -Pc.view(-1)[::3]
                P.copy_(Pc)
                Po[li] = np.ascontiguousarray(to_np(P))
            ctx.params_changed()
        if side_stream:
            # a caller's non-blocking stream (every torch side stream is one): the library's
            # host->device uploads must be ordered on it, not on the legacy default stream
            ss = torch.cuda.Stream()
            ss.wait_stream(torch.cuda.current_stream())
            ctx.step(t, Gs, Ps, stream=ss)
            ctx.sync()
            ss.synchronize()
        else:
            ctx.step(t, Gs, Ps)
            ctx.sync()
        warm = t < warmup
        refresh = not warm and (t - warmup) % N == 0
        for li, (n, m) in enumerate(shapes):
            L = layers[li]
            gidx = to_np(ctx.selected(li))
            if refresh:
                # lagged selection (R24): a refresh after the first ranks by the previous step's
                # norms; after a step that is also a pre-refresh step (N = 1) the norms buffer
                # already holds this step's
                lag = lagged and L.lag_norms is not None
                onorms = orc.column_norms(prevG[li] if lag else Gn[li])
                pre_now = lagged and (t - warmup + 1) % N == 0
                if not pre_now:
                    assert_close_rel(to_np(ctx.norms(li)), onorms, 1e-5, f"norms t={t} l={li}")
                swaps += selection_ok(gidx, orc.topk(onorms, L.k), onorms)
            out = L.step(t, Gn[li], Po[li], idx_override=gidx if refresh else None)
            if t % check_every and t != steps - 1:
                continue
            assert_bits_equal(gidx, L.idx, f"idx t={t} l={li}")
            M, V, st = ctx.optimizer_state(li)
            assert_bits_equal(to_np(st), L.steps, f"steps t={t} l={li}")
            assert_bits_equal(to_np(M), L.M, f"exp_avg t={t} l={li}")
            assert_bits_equal(to_np(V), L.V, f"exp_avg_sq t={t} l={li}")
            assert_bits_equal(np.ascontiguousarray(to_np(Ps[li])), Po[li], f"params t={t} l={li}")
            if warm:
                assert out.shape == (n, 0)
                continue
            assert_bits_equal(to_np(ctx.compact_buffer(li)), out, f"compact t={t} l={li}")
            if offload and devacc:
                assert ctx.compact_host(li) is None and ctx.host_accumulator(li, 0) is None
                assert_bits_equal(to_np(ctx.device_accumulator(li, 0)), L.acc[((t - warmup) // S) % 2],
                                  f"device acc t={t} l={li}")
            elif offload:
                assert_bits_equal(ctx.compact_host(li).copy(), out, f"compact host t={t} l={li}")
                assert_bits_equal(ctx.host_accumulator(li, 0).copy(), L.acc[((t - warmup) // S) % 2], f"acc t={t} l={li}")
            if offload:
                sealed = ctx.host_accumulator(li, 1)
                osealed = L.sealed(t)
                assert (sealed is None) == (osealed is None)
                if sealed is not None:
                    assert_bits_equal(sealed.copy(), osealed, f"sealed acc t={t} l={li}")
        prevG = Gn
    launches = ctx.kernel_launches()
    ctx.close()
    return swaps, launches


@pytest.mark.parametrize("NS", [1, 2, 4])
def test_step_config1_fp32(zf, orc, gpu, NS):
    """BASELINE config 1: one 256x512 fp32 gradient, top-10%, selective AdamW +
    unselected accumulation; N = S in {1, 2, 4}, 8 steps (two windows at S=4)."""
    swaps, launches = _run_stateful(zf, orc, gpu, [(256, 512)], "fp32", "fp32", 100000, NS, NS, 8, offload=True)
    # per step: K3 prologue + K3; per refresh: K1 + K2; plus a table patch (k_patch) whenever
    # a step's launch table differs from what the device holds (at most norm + update table)
    base = 2 * 8 + 2 * (8 // NS)
    assert base <= launches <= base + 2 * 8, launches
    assert swaps == 0


@pytest.mark.parametrize("NS,pdt,wd", [(1, "fp32", 0.0), (2, "fp32", 0.01), (4, "fp32", 0.0), (4, "bf16", 0.0),
                                      (2, "bf16", 0.01)])
def test_step_cpu_update(zf, orc, gpu, NS, pdt, wd):
    """f1 (reading R18): the unselected columns take one AdamW step per window on the host
    fp32 master with the window's average gradient; parameters bit-exact against the
    oracle's deferred update, including migration at refreshes."""
    swaps, launches = _run_stateful(zf, orc, gpu, [(256, 512), (37, 1001)], "bf16" if pdt == "bf16" else "fp32",
                                    pdt, 100000, NS, NS, 9, offload=True, wd=wd, cpu_update=True)
    # K1+K2 per refresh, K3 per step, K5 per layer per window end, plus K5' gathers of entering columns
    assert launches >= 9 + 2 * len(range(0, 9, NS)) + 2 * (9 // NS) + 2
    assert swaps == 0


@pytest.mark.parametrize("tau,NS,pdt,cpu", [(1, 2, "bf16", False), (3, 2, "fp32", False), (2, 4, "bf16", True),
                                           (5, 1, "fp32", True)])
def test_step_warmup(zf, orc, gpu, tau, NS, pdt, cpu):
    """f2 warm-up (reading R20): tau synchronous steps with k = m (moments [n, m]), then the
    regular schedule from step tau with the R7 remap out of the all-columns set; selection,
    moments, step counts, params, compact blocks and accumulators bit-exact vs the oracle."""
    shapes = [(64, 512), (37, 1001), (16, 4096)]
    gdt = "bf16" if pdt == "bf16" else "fp32"
    _run_stateful(zf, orc, gpu, shapes, gdt, pdt, 100000, NS, NS, tau + 6, offload=True, cpu_update=cpu,
                  warmup=tau)


@pytest.mark.parametrize("lagged", [False, True])
def test_step_nccl_one_rank(zf, orc, gpu, lagged):
    """The NCCL exchange path on one GPU: world 1 with an NCCL id makes a one-rank
    communicator, so every refresh runs ncclAllReduce on the flat norm vector (on the
    caller's stream, or the side stream with the lagged selection) -- the multi-GPU code
    path, exercised here; results bit-exact with the oracle, norms rel 1e-5."""
    real = zf.Context
    nid = zf.zf_nccl_unique_id()
    try:
        zf.Context = lambda *a, **kw: real(*a, nccl_id=nid, **kw)
        _run_stateful(zf, orc, gpu, [(96, 320), (64, 512)], "bf16", "bf16", 100000, 2, 2, 6, offload=True,
                      lagged=lagged)
    finally:
        zf.Context = real


@pytest.mark.parametrize("shapes,gdt,NS,cpu", [([(512, 1024), (96, 320), (0, 512), (37, 1001), (640, 1024), (64, 512)],
                                                "bf16", 2, False),
                                               ([(512, 1024), (130, 257), (700, 900)], "fp32", 4, True)])
def test_step_refresh_in_groups(zf, orc, gpu, shapes, gdt, NS, cpu):
    """f4 (i): refresh steps run K1 -> K2 -> K3 per group of layers (1-MB groups: single
    layers and runs of small ones, a layer without rows among them) -- the unit ranges of
    each launch offset to its group; everything bit-exact with the oracle."""
    _run_stateful(zf, orc, gpu, shapes, gdt, gdt, 100000, NS, NS, 3 * NS + 1, offload=True, cpu_update=cpu,
                  refresh_group_mb=1)


def test_refresh_groups_argument_errors(zf):
    with pytest.raises(zf.ZFError):
        zf.Context([zf.LayerShape(8, 64)], topk_ratio_ppm=100000, refresh_interval=2, accum_interval=2,
                   refresh_group_mb=-1)
    with pytest.raises(zf.ZFError):
        zf.Context([zf.LayerShape(8, 64)], topk_ratio_ppm=100000, refresh_interval=2, accum_interval=2,
                   refresh_group_mb=8, lagged_selection=True)


def test_nccl_one_rank_contexts_in_sequence(zf, orc, gpu):
    """Several contexts one after another, each with its own NCCL id (an id bootstraps one
    communicator; bench.py makes a fresh one per context), each bit-exact."""
    real = zf.Context
    try:
        zf.Context = lambda *a, **kw: real(*a, nccl_id=zf.zf_nccl_unique_id(), **kw)
        for _ in range(3):
            _run_stateful(zf, orc, gpu, [(64, 512)], "bf16", "bf16", 100000, 2, 2, 3, offload=False)
    finally:
        zf.Context = real


@pytest.mark.parametrize("host_stages", [2, 4])
def test_step_x1_many_chunks(zf, orc, gpu, monkeypatch, host_stages):
    """X1 with 16-KB chunks (ZF_X1_CHUNK_KB): many chunks, each gated by its own K3
    completion counter and copied by the X1 thread, layers without rows among them; the host
    compact blocks, both accumulators and everything else bit-exact."""
    monkeypatch.setenv("ZF_X1_CHUNK_KB", "16")
    shapes = [(0, 512), (37, 1001), (96, 300), (0, 4096), (64, 512), (130, 257), (0, 77), (20, 2000)]
    _run_stateful(zf, orc, gpu, shapes, "bf16", "bf16", 100000, 2, 2, 6, offload=True, host_stages=host_stages)


@pytest.mark.parametrize("shapes,gdt,NS,tau,cpu", [([(256, 512)], "fp32", 2, 0, False),
                                                  ([(64, 512), (37, 1001), (16, 4096)], "bf16", 2, 2, True),
                                                  ([(513, 768), (64, 4096)], "bf16", 4, 0, False)])
def test_step_state_offload(zf, orc, gpu, shapes, gdt, NS, tau, cpu):
    """f3 state swap-out: moments in mapped pinned host memory, streamed by K3 over
    the host link; every result bit-identical to the oracle (and so to the HBM-resident path)."""
    _run_stateful(zf, orc, gpu, shapes, gdt, gdt, 100000, NS, NS, tau + 5, offload=True, cpu_update=cpu,
                  warmup=tau, state_offload=True)


@pytest.mark.parametrize("shapes,offload", [([(0, 512), (37, 1001), (0, 4096), (64, 512), (0, 77)], True),
                                            ([(33, 300), (0, 777)], True), ([(33, 33), (0, 1025)], False)])
@pytest.mark.parametrize("cpu", [False, True])
def test_step_layers_without_rows(zf, orc, gpu, shapes, offload, cpu):
    """Flat partitions (row f3): matrices with no rows on this rank (n = 0) ride along --
    zero norms, the same selection rule, nothing else -- while the others stay bit-exact.
    A rows-less LAST layer's empty views sit at the end of the library's blocks (found by the
    600-seed random soak, `profiles/r02ao_pytest_random600.log`)."""
    _run_stateful(zf, orc, gpu, shapes, "bf16", "bf16", 100000, 2, 2, 5, offload=offload,
                  cpu_update=cpu and offload)


@pytest.mark.parametrize("shapes,gdt,NS,tau,cpu", [([(256, 512)], "fp32", 2, 0, False),
                                                  ([(64, 512), (37, 1001), (0, 96), (16, 4096)], "bf16", 2, 1, True),
                                                  ([(513, 768), (64, 4096)], "bf16", 4, 0, True),
                                                  ([(130, 257), (5, 20000)], "fp32", 1, 0, False)])
def test_step_device_accumulate(zf, orc, gpu, shapes, gdt, NS, tau, cpu):
    """K7 (device_accumulate): the window accumulators live in HBM and only sealed windows go
    to the host; device active accumulator, host sealed copy, f1 updates bit-exact."""
    _run_stateful(zf, orc, gpu, shapes, gdt, gdt, 100000, NS, NS, tau + 7, offload=True, cpu_update=cpu,
                  warmup=tau, devacc=True)


@pytest.mark.parametrize("ppm", [1000000, 1])
def test_step_degenerate_k(zf, orc, gpu, ppm):
    """k = m (every column important: plain AdamW, empty compact block) and k = 1."""
    shapes = [(64, 512), (37, 1001)]
    _run_stateful(zf, orc, gpu, shapes, "bf16", "bf16", ppm, 2, 2, 4, offload=True, cpu_update=True)
    _run_stateful(zf, orc, gpu, shapes, "fp32", "fp32", ppm, 2, 2, 3, offload=True, devacc=True)


def test_zen_auto_gpu_spec_worked_example(zf):
    """SPEC S:434 on the GPU, against the closed form (not the oracle): a constant stream whose
    unimportant per-channel norm is 0.25 x the important one triggers the window end at the
    4th step with gamma = 1 (windows of 4 steps; refresh every 16)."""
    n, m = 64, 256
    k = zf.k_for(m, 100000)
    G = torch.full((n, m), 0.25, dtype=torch.bfloat16, device="cuda")
    G[:, :k] = 1.0
    P = torch.zeros(n, m, dtype=torch.bfloat16, device="cuda")
    ctx = zf.Context([zf.LayerShape(n, m)], topk_ratio_ppm=100000, refresh_interval=16, accum_interval=16,
                     offload=True, host_accumulate=True, auto_gamma=1.0)
    for t in range(16):
        ctx.step(t, [G], [P])
    ctx.sync()
    log = ctx.window_log()
    ctx.close()
    assert [t for (t, e, *_r) in log if e] == [3, 7, 11, 15]
    for t, e, A, i, u in log:
        assert abs(u / i - 0.25) < 1e-6 and abs(A - ((t % 4) + 1) * u) <= 1e-9 * A


@pytest.mark.parametrize("NS,pdt,devacc", [(2, "bf16", False), (4, "fp32", True), (1, "bf16", True)])
def test_step_cpu_update_async(zf, orc, gpu, NS, pdt, devacc):
    """R23: the window-end CPU AdamW runs on a worker thread and lands at the next zf_step /
    zf_sync -- after every zf_sync the state is bit-exact with the oracle's synchronous f1."""
    gdt = "bf16" if pdt == "bf16" else "fp32"
    _run_stateful(zf, orc, gpu, [(256, 512), (37, 1001)], gdt, pdt, 100000, NS, NS, 9, offload=True,
                  cpu_update=True, cpu_async=True, devacc=devacc)


@pytest.mark.parametrize("cpu_async", [False, True])
def test_step_cpu_update_on_a_side_stream(zf, orc, gpu, cpu_async):
    """f1 with zf_step on a non-blocking torch stream: the refresh's column-list uploads and
    the K5 scatter are ordered on the caller's stream (bit-exact vs the oracle)."""
    _run_stateful(zf, orc, gpu, [(96, 300), (64, 128)], "bf16", "bf16", 100000, 2, 2, 7, offload=True,
                  cpu_update=True, cpu_async=cpu_async, side_stream=True)


@pytest.mark.parametrize("shapes,gdt,NS,cpu", [([(256, 512)], "fp32", 4, False), ([(300, 4096), (64, 1000)], "bf16", 2, True),
                                              ([(96, 11008), (40, 4096)], "bf16", 4, False)])
def test_step_param_subset_off(zf, orc, gpu, shapes, gdt, NS, cpu):
    """param_subset = 0 (p's selected values read from p on every step) is bit-exact too."""
    _run_stateful(zf, orc, gpu, shapes, gdt, gdt, 100000, NS, NS, 9, offload=True, cpu_update=cpu, psub=False)


@pytest.mark.parametrize("shapes,gdt,pdt,NS,cpu,psub", [([(256, 512)], "fp32", "fp32", 4, False, True),
                                                   ([(300, 4096), (64, 1000)], "bf16", "bf16", 2, True, True),
                                                   ([(96, 4096), (40, 700)], "bf16", "fp32", 4, False, False)])
def test_step_split_update(zf, orc, gpu, monkeypatch, shapes, gdt, pdt, NS, cpu, psub):
    """The split update (ZF_K3_SPLIT: K3a compaction + extraction, K3b dense AdamW over the
    [n, k] blocks, incl. the moment remap and the branch-free division/sqrt fast path) is
    bit-exact vs the oracle as well."""
    monkeypatch.setenv("ZF_K3_SPLIT", "1")
    _run_stateful(zf, orc, gpu, shapes, gdt, pdt, 100000, NS, NS, 9, offload=True, cpu_update=cpu, psub=psub)


@pytest.mark.parametrize("shapes,gdt,NS,cpu,warmup", [([(256, 512)], "fp32", 4, False, 0),
                                                      ([(300, 4096), (64, 1000)], "bf16", 2, True, 0),
                                                      ([(96, 700), (40, 256)], "bf16", 1, False, 0),
                                                      ([(128, 1024)], "bf16", 2, True, 3)])
def test_step_lagged_selection(zf, orc, gpu, shapes, gdt, NS, cpu, warmup):
    """f4 (ii), reading R24: a refresh after the first selects by the previous step's norms (K1
    on the side stream at the end of the pre-refresh step); selection bit-exact on those norms,
    everything downstream bit-exact vs the oracle's lagged mode (N = S in {1, 2, 4}, f1, warm-up)."""
    _run_stateful(zf, orc, gpu, shapes, gdt, gdt, 100000, NS, NS, 9 + warmup, offload=True, cpu_update=cpu,
                  warmup=warmup, lagged=True)


def test_lagged_selection_needs_fixed_windows(zf):
    with pytest.raises(zf.ZFError):
        zf.Context([zf.LayerShape(8, 64)], offload=True, host_accumulate=True, auto_gamma=0.5,
                   lagged_selection=True)


@pytest.mark.parametrize("poke", [{2, 5, 6}, {4, 8}])
@pytest.mark.parametrize("ppm", [100000, 10000])
def test_params_changed_rereads_the_selected_columns(zf, orc, gpu, ppm, poke):
    """param_subset: the caller rewrites p between refreshes (t = 2, 5, 6) or right before a
    refresh (t = 4, 8: that refresh must read p, not the previous subset block) and calls
    zf_params_changed; the next steps use the new values (bit-exact vs the oracle, which sees
    the same writes)."""
    _run_stateful(zf, orc, gpu, [(128, 4096), (96, 700)], "bf16", "bf16", ppm, 4, 4, 9, offload=False,
                  poke=poke)


def test_cpu_update_async_is_stale_until_the_next_call(zf, gpu):
    """Between a window's last zf_step and the next call, the unselected columns still hold
    their pre-update values (the one-window staleness of the overlapped update); the next
    zf_step applies the update before anything else."""
    n, m = 64, 512
    ctx = zf.Context([zf.LayerShape(n, m)], topk_ratio_ppm=100000, refresh_interval=2, accum_interval=2,
                     offload=True, host_accumulate=True, cpu_update=True, cpu_update_async=True)
    G = _grad(gpu, n, m, "bf16")
    P = torch.zeros(n, m, dtype=torch.bfloat16, device="cuda")
    ctx.step(0, [G], [P])
    ctx.step(1, [G], [P])                      # window end: CPU update launched, not applied
    torch.cuda.synchronize()
    unsel = torch.ones(m, dtype=torch.bool, device="cuda")
    unsel[ctx.selected(0).long()] = False
    assert torch.all(P[:, unsel] == 0)
    ctx.sync()                                 # lands the update
    assert torch.count_nonzero(P[:, unsel]) > 0
    ctx.close()


def test_step_lr_schedule(zf, orc, gpu):
    """zf_set_lr (a schedule): the bias-corrected step size of the next step uses the
    new lr, on the GPU (K3) and in the deferred CPU update; bit-exact vs the oracle run with
    the same per-step lr (decoupled weight decay uses it too)."""
    shapes = [(64, 512), (37, 1001)]
    hp = orc.AdamHP(lr=1e-3, weight_decay=0.01)
    ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], grad_dtype=torch.bfloat16, param_dtype=torch.float32,
                     topk_ratio_ppm=100000, refresh_interval=2, accum_interval=2,
                     adam=zf.adam_params(lr=1e-3, weight_decay=0.01), offload=True, host_accumulate=True,
                     cpu_update=True)
    scales = [gpu.ColScale(m, li) for li, (n, m) in enumerate(shapes)]
    Gs = [torch.empty(n, m, dtype=torch.bfloat16, device="cuda") for n, m in shapes]
    Ps = [torch.empty(n, m, dtype=torch.float32, device="cuda") for n, m in shapes]
    for li, P in enumerate(Ps):
        gpu.fill_param(P, li)
    layers = [orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=2, accum_interval=2, hp=hp,
                              cpu_update=True) for n, m in shapes]
    Po = [to_np(P) for P in Ps]
    for t in range(6):
        lr = 1e-3 * (0.5 ** t)
        ctx.set_lr(lr)
        hp.lr = lr
        for li, (G, sc) in enumerate(zip(Gs, scales)):
            sc.advance_to(t)
            gpu.fill_grad(G, li, t, sc)
        ctx.step(t, Gs, Ps)
        ctx.sync()
        for li, L in enumerate(layers):
            gidx = to_np(ctx.selected(li))
            L.step(t, to_np(Gs[li]), Po[li], idx_override=gidx if t % 2 == 0 else None)
            assert_bits_equal(to_np(Ps[li]), Po[li], f"params t={t} l={li}")
    ctx.close()


def test_profile_phases(zf, gpu):
    """zf_profile / zf_profile_read: per-phase event timings and counts (K1 and K2 on refresh
    steps, K3 every step, the per-step D2H span with offload; K7 and the window D2H with
    device accumulation)."""
    G = _grad(gpu, 256, 512, "bf16")
    P = torch.zeros(256, 512, dtype=torch.bfloat16, device="cuda")
    for devacc in (False, True):
        ctx = zf.Context([zf.LayerShape(256, 512)], topk_ratio_ppm=100000, refresh_interval=2, accum_interval=2,
                         offload=True, host_accumulate=True, device_accumulate=devacc)
        ctx.profile(True)
        for t in range(4):
            ctx.step(t, [G], [P])
        ctx.sync()
        prof = ctx.profile_read()
        ctx.close()
        assert prof["k1_norms"][1] == 2 and prof["k2_topk"][1] == 2 and prof["k3_update"][1] == 4
        assert prof["allreduce"][1] == 0
        if devacc:
            assert prof["k7_accumulate"][1] == 4 and prof["d2h_window"][1] == 2 and prof["d2h_step"][1] == 0
        else:
            assert prof["d2h_step"][1] == 4 and prof["k7_accumulate"][1] == 0
        assert all(ms >= 0.0 for ms, _n in prof.values()) and prof["k3_update"][0] > 0.0


def test_step_paper_lr_most_values_unchanged(zf, orc, gpu):
    """At the paper's lr 1e-5 most bf16 parameters keep their bits in a step; K3 stores only
    changed values (reading the staged tile) -- parameters, moments, compaction and
    accumulators must still be bit-exact (staged-p and unstaged-p layers, f1 on)."""
    shapes = [(64, 4096), (130, 257), (33, 1000)]
    _run_stateful(zf, orc, gpu, shapes, "bf16", "bf16", 100000, 2, 2, 5, offload=True, lr=1e-5, cpu_update=True)
    _run_stateful(zf, orc, gpu, shapes, "bf16", "bf16", 10000, 2, 2, 4, offload=True, lr=1e-5)


def test_cpu_update_needs_aligned_windows(zf):
    with pytest.raises(zf.ZFError):
        zf.Context([zf.LayerShape(8, 64)], refresh_interval=2, accum_interval=4, offload=True, host_accumulate=True,
                   cpu_update=True)


def test_step_config1_weight_decay(zf, orc, gpu):
    _run_stateful(zf, orc, gpu, [(256, 512)], "fp32", "fp32", 100000, 4, 4, 6, offload=True, wd=0.01)


def test_step_ragged_multilayer_bf16(zf, orc, gpu):
    shapes = [(37, 1001), (513, 768), (130, 257), (5, 20000), (1, 64), (64, 4096)]
    _run_stateful(zf, orc, gpu, shapes, "bf16", "bf16", 100000, 2, 2, 5, offload=True, ld_pad=8)


def test_step_tie_heavy(zf, orc, gpu):
    _run_stateful(zf, orc, gpu, [(64, 1000), (16, 333)], "bf16", "bf16", 10000, 2, 2, 4, offload=False, tie=True)


def test_step_gpt2_small_bf16(zf, orc, gpu):
    """BASELINE config 2: GPT-2 small, all 49 linears, bf16, k=10%, N=4 (refresh at 0 and 4)."""
    shapes = [(n, m) for _, n, m in synth.gpt2_small_linears()]
    _run_stateful(zf, orc, gpu, shapes, "bf16", "bf16", 100000, 4, 4, 5, offload=False, check_every=4)


def test_step_nonfinite_reported(zf, gpu):
    ctx = zf.Context([zf.LayerShape(64, 512)], topk_ratio_ppm=100000, refresh_interval=2, accum_interval=2)
    G = _grad(gpu, 64, 512, "bf16")
    P = torch.zeros(64, 512, dtype=torch.bfloat16, device="cuda")
    ctx.step(0, [G], [P])
    ctx.sync()
    G[3, 5] = float("inf")
    ctx.step(1, [G], [P])
    with pytest.raises(zf.ZFError) as e:
        ctx.sync()
    assert e.value.status == zf.ZF_ENONFINITE
    ctx.step(2, [_grad(gpu, 64, 512, "bf16")], [P])
    ctx.sync()  # flag cleared
    ctx.close()


@pytest.mark.parametrize("dt", ["bf16", "fp32"])
@pytest.mark.parametrize("where", ["selected", "unselected"])
@pytest.mark.parametrize("bad", [float("inf"), float("nan")])
def test_step_nonfinite_on_a_steady_step(zf, gpu, dt, where, bad):
    """Steady steps run no K1: a non-finite gradient must be caught by K3 itself -- by its
    AdamW (a selected column) or by its compaction (an unselected one) -- and reported by
    zf_sync as ZF_ENONFINITE (SPEC S:44 / S:266, reading R15)."""
    n, m = 64, 512
    ctx = zf.Context([zf.LayerShape(n, m)], grad_dtype=TDT[dt], param_dtype=TDT[dt], topk_ratio_ppm=100000,
                     refresh_interval=4, accum_interval=4)
    G = _grad(gpu, n, m, dt)
    P = torch.zeros(n, m, dtype=TDT[dt], device="cuda")
    ctx.step(0, [G], [P])
    ctx.sync()
    sel = set(to_np(ctx.selected(0)).tolist())
    col = sorted(sel)[3] if where == "selected" else next(j for j in range(m) if j not in sel)
    G2 = G.clone()
    G2[7, col] = bad
    ctx.step(1, [G2], [P])
    with pytest.raises(zf.ZFError) as e:
        ctx.sync()
    assert e.value.status == zf.ZF_ENONFINITE
    ctx.close()


def test_lagged_refresh_waits_for_the_side_stream_norms(zf, orc, monkeypatch):
    """f4 (ii): the refresh step must wait for the previous step's side-stream K1.  The test
    knob ZF_TEST_LAG_DELAY_US holds the side stream 50 ms before every lagged K1, the steps
    are enqueued back to back without zf_sync (gradients resident, as the contract asks), and
    every step's gradient ranks different columns first; selection, parameters and moments
    after six steps (refreshes at 0, 2, 4) must equal the oracle's."""
    monkeypatch.setenv("ZF_TEST_LAG_DELAY_US", "50000")
    n, m, N, T = 64, 512, 2, 6
    rng = np.random.default_rng(11)
    Gh = [(rng.standard_normal((n, m)) * rng.permutation(np.geomspace(1e-3, 1.0, m))[None, :]).astype(np.float32)
          for _ in range(T)]
    Gd = [torch.from_numpy(g).cuda() for g in Gh]
    P = torch.zeros(n, m, device="cuda")
    Po = np.zeros((n, m), np.float32)
    ctx = zf.Context([zf.LayerShape(n, m)], grad_dtype=torch.float32, param_dtype=torch.float32,
                     topk_ratio_ppm=100000, refresh_interval=N, accum_interval=N, lagged_selection=True)
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=N, accum_interval=N, lagged=True)
    torch.cuda.synchronize()
    for t in range(T):
        ctx.step(t, [Gd[t]], [P])
    ctx.sync()
    for t in range(T):
        L.step(t, Gh[t], Po)
    Md, Vd, sd = ctx.optimizer_state(0)
    assert_bits_equal(to_np(ctx.selected(0)), L.idx, "idx")
    assert_bits_equal(to_np(sd), L.steps, "steps")
    assert_bits_equal(to_np(Md), L.M, "exp_avg")
    assert_bits_equal(to_np(Vd), L.V, "exp_avg_sq")
    assert_bits_equal(np.ascontiguousarray(to_np(P)), Po, "params")
    ctx.close()


def test_step_state_errors(zf, gpu):
    ctx = zf.Context([zf.LayerShape(8, 64)], refresh_interval=4, accum_interval=4)
    G = _grad(gpu, 8, 64, "bf16")
    P = torch.zeros(8, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(zf.ZFError) as e:
        ctx.step(1, [G], [P])            # first step must refresh
    assert e.value.status == zf.ZF_ESTATE
    ctx.step(0, [G], [P])
    with pytest.raises(zf.ZFError):
        ctx.step(2, [G], [P])            # not consecutive
    ctx.close()


# ------------------------------------------------------------------ full-size configs (sampled)
def _run_fullsize(zf, orc, gpu, names, ppm, steps, sample, offload, row_div=1, lr=1e-5):
    """Whole model through zf_step in the bench launch configuration; the sampled
    layers are checked against the oracle one by one (bf16 G and p, fp32 state)."""
    shapes = [(n // row_div, m) for _, n, m in names]
    ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], topk_ratio_ppm=ppm, refresh_interval=4,
                     accum_interval=4, adam=zf.adam_params(lr=lr), offload=offload, host_accumulate=offload)
    hp_o = orc.AdamHP(lr=lr)
    tot = sum(n * m for n, m in shapes)
    gbuf = torch.empty(tot, dtype=torch.bfloat16, device="cuda")
    pbuf = torch.empty(tot, dtype=torch.bfloat16, device="cuda")
    Gs, Ps, off = [], [], 0
    for n, m in shapes:
        Gs.append(gbuf[off:off + n * m].view(n, m))
        Ps.append(pbuf[off:off + n * m].view(n, m))
        off += n * m
    scales = [gpu.ColScale(m, li) for li, (n, m) in enumerate(shapes)]
    for li, P in enumerate(Ps):
        gpu.fill_param(P, li)
    layers = {li: orc.OracleLayer(n=shapes[li][0], m=shapes[li][1], ratio_ppm=ppm, refresh_interval=4,
                                  accum_interval=4, hp=hp_o) for li in sample}
    Po = {li: to_np(Ps[li]) for li in sample}
    for t in range(steps):
        for li, (G, sc) in enumerate(zip(Gs, scales)):
            sc.advance_to(t)
            gpu.fill_grad(G, li, t, sc)
        Gn = {li: to_np(Gs[li]) for li in sample}
        ctx.step(t, Gs, Ps)
        ctx.sync()
        for li in sample:
            L = layers[li]
            gidx = to_np(ctx.selected(li))
            if t % 4 == 0:
                onorms = orc.column_norms(Gn[li])
                assert_close_rel(to_np(ctx.norms(li)), onorms, 1e-5, f"norms t={t} l={li}")
                selection_ok(gidx, orc.topk(onorms, L.k), onorms)
            out = L.step(t, Gn[li], Po[li], idx_override=gidx if t % 4 == 0 else None)
            M, V, st = ctx.optimizer_state(li)
            assert_bits_equal(to_np(st), L.steps, f"steps t={t} l={li}")
            assert_bits_equal(to_np(M), L.M, f"exp_avg t={t} l={li}")
            assert_bits_equal(to_np(V), L.V, f"exp_avg_sq t={t} l={li}")
            assert_bits_equal(to_np(Ps[li]), Po[li], f"params t={t} l={li}")
            assert_bits_equal(to_np(ctx.compact_buffer(li)), out, f"compact t={t} l={li}")
            if offload:
                assert_bits_equal(ctx.compact_host(li).copy(), out, f"compact host t={t} l={li}")
                assert_bits_equal(ctx.host_accumulator(li, 0).copy(), L.acc[(t // 4) % 2], f"acc t={t} l={li}")
    ctx.close()


@pytest.mark.slow
def test_llama2_7b_fullsize_sampled(zf, orc, gpu):
    """BASELINE config 3 at full size (225 linears, 6.6 G elements, k=10%), refresh at
    t=0 then a steady step; q_proj, gate_proj, down_proj of layer 0 and lm_head checked."""
    _run_fullsize(zf, orc, gpu, synth.llama2_7b_linears(), 100000, 2, [0, 4, 6, 224], offload=False)


@pytest.mark.slow
def test_llama2_7b_fullsize_k1pct_sampled(zf, orc, gpu):
    """BASELINE config 3 at k = 1% (225 linears, 6.6 G elements; k = 41 / 111 per matrix), in
    the bench's launch configuration, over two refreshes (t = 0 and 4) and the steady steps
    between them; q_proj, gate_proj, down_proj of layer 0 and lm_head checked."""
    _run_fullsize(zf, orc, gpu, synth.llama2_7b_linears(), 10000, 5, [0, 4, 6, 224], offload=False)


@pytest.mark.slow
def test_llama2_13b_rank0_shard_offload_sampled(zf, orc, gpu):
    """BASELINE config 5 on one GPU: the row shard rank 0 of 8 would own (n/8 rows of all
    281 linears), k=10%, with D2H offload + host accumulation; sampled layers checked."""
    _run_fullsize(zf, orc, gpu, synth.llama2_13b_linears(), 100000, 2, [0, 5, 6, 280], offload=True, row_div=8)


# ------------------------------------------------------------------ f2: Zen-auto (reading R21)
def _run_auto(zf, orc, gpu, shapes, gdt, pdt, ppm, N, smax, gamma, steps, cpu_update=False, warmup=0, lr=1e-3,
              devacc=False):
    """zf_step with auto_gamma against OracleModel: per step the window decision and its
    inputs (A, mean important / unimportant channel norm), and bit for bit the selection,
    moments, parameters (incl. f1 updates with the window's length), compact blocks and
    both host accumulators."""
    hp_o = orc.AdamHP(lr=lr)
    ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], grad_dtype=TDT[gdt], param_dtype=TDT[pdt],
                     topk_ratio_ppm=ppm, refresh_interval=N, accum_interval=smax, adam=zf.adam_params(lr=lr),
                     offload=True, host_accumulate=True, cpu_update=cpu_update, warmup_steps=warmup,
                     auto_gamma=gamma, device_accumulate=devacc)
    scales = [gpu.ColScale(m, li) for li, (n, m) in enumerate(shapes)]
    Gs = [torch.empty(n, m, dtype=TDT[gdt], device="cuda") for n, m in shapes]
    Ps = [torch.empty(n, m, dtype=TDT[pdt], device="cuda") for n, m in shapes]
    for li, P in enumerate(Ps):
        gpu.fill_param(P, li)
    model = orc.OracleModel([orc.OracleLayer(n=n, m=m, ratio_ppm=ppm, refresh_interval=N, accum_interval=smax,
                                             hp=hp_o, cpu_update=cpu_update, warmup=warmup) for n, m in shapes],
                            auto_gamma=gamma)
    Po = [np.ascontiguousarray(to_np(P)) for P in Ps]
    sealed_buf = None
    for t in range(steps):
        for li, (G, sc) in enumerate(zip(Gs, scales)):
            sc.advance_to(t)
            gpu.fill_grad(G, li, t, sc)
        Gn = [np.ascontiguousarray(to_np(G)) for G in Gs]
        ctx.step(t, Gs, Ps)
        ctx.sync()
        refresh = t >= warmup and (t - warmup) % N == 0
        ov = None
        if refresh:
            ov = []
            for li, L in enumerate(model.layers):
                gidx = to_np(ctx.selected(li))
                onorms = orc.column_norms(Gn[li])
                assert selection_ok(gidx, orc.topk(onorms, L.k), onorms) == 0
                ov.append(gidx)
        w_before = model.w
        model.step(t, Gn, Po, idx_overrides=ov)
        for li, L in enumerate(model.layers):
            assert_bits_equal(to_np(ctx.selected(li)), L.idx, f"idx t={t} l={li}")
            M, V, st = ctx.optimizer_state(li)
            assert_bits_equal(to_np(M), L.M, f"exp_avg t={t} l={li}")
            assert_bits_equal(to_np(V), L.V, f"exp_avg_sq t={t} l={li}")
            assert_bits_equal(np.ascontiguousarray(to_np(Ps[li])), Po[li], f"params t={t} l={li}")
        if t < warmup:
            continue
        log = ctx.window_log()
        lt, lend, lA, li_, lu = log[-1]
        oA, oi, ou = model.stats[-1]
        assert lt == t and len(log) == t - warmup + 1
        assert abs(oA - gamma * oi) > 1e-4 * gamma * oi, "decision too close to call (pick another gamma)"
        assert lend == (model.ends[-1:] == [t]), f"window decision t={t}"
        for got, want, what in ((lA, oA, "A"), (li_, oi, "imp"), (lu, ou, "unimp")):
            assert abs(got - want) <= 1e-5 * abs(want), (t, what, got, want)
        for li, L in enumerate(model.layers):
            got = to_np(ctx.device_accumulator(li, 0)) if devacc else ctx.host_accumulator(li, 0).copy()
            assert_bits_equal(got, L.acc[w_before % 2], f"acc t={t} l={li}")
        if lend:
            sealed_buf = w_before % 2
        for li, L in enumerate(model.layers):
            s = ctx.host_accumulator(li, 1)
            assert (s is None) == (sealed_buf is None)
            if s is not None:
                assert_bits_equal(s.copy(), L.acc[sealed_buf], f"sealed acc t={t} l={li}")
    ends = [e for (e, end, *_r) in ctx.window_log() if end]
    ctx.close()
    assert ends == model.ends
    return model.intervals()


AUTO_SHAPES = [(64, 256), (96, 200), (128, 320)]


@pytest.mark.parametrize("gamma,cpu,pdt,devacc", [(0.15, False, "bf16", False), (0.15, True, "bf16", False),
                                                  (0.25, True, "fp32", False), (0.1, False, "fp32", False),
                                                  (0.15, False, "bf16", True), (0.25, True, "bf16", True)])
def test_step_zen_auto(zf, orc, gpu, gamma, cpu, pdt, devacc):
    """Zen-auto (f2, reading R21) on column-concentrated synthetic gradients: intervals vary
    (not all equal to S_max), windows cut at the refresh every 8 steps."""
    gdt = "bf16" if pdt == "bf16" else "fp32"
    iv = _run_auto(zf, orc, gpu, AUTO_SHAPES, gdt, pdt, 100000, 8, 8, gamma, 16, cpu_update=cpu, devacc=devacc)
    assert sum(iv) == 16 and min(iv) < 8, iv


def test_step_zen_auto_cap_refresh_and_warmup(zf, orc, gpu):
    """S_max (= accum_interval) and the refresh boundary cut windows; the schedule starts after
    tau warm-up steps."""
    iv = _run_auto(zf, orc, gpu, AUTO_SHAPES, "bf16", "bf16", 100000, 6, 3, 0.5, 14, cpu_update=True, warmup=2)
    assert max(iv) <= 3 and sum(iv) == 12, iv


# ------------------------------------------------------------------ H1 in window batches (host_stages)
@pytest.mark.parametrize("host_stages,S,N,gdt,cpu", [(8, 4, 8, "bf16", False), (3, 4, 8, "bf16", True),
                                                     (2, 2, 4, "bf16", False), (6, 4, 8, "fp32", False),
                                                     (16, 8, 8, "bf16", True)])
def test_h1_window_batches(zf, orc, gpu, host_stages, S, N, gdt, cpu):
    """H1 (row a8) accumulating several staged steps of a window in one pass: steps are issued
    without a zf_sync inside a window, so H1 finds several staged steps (batches of up to
    host_stages, never across a window end); the active and sealed accumulators, the f1
    parameters and the window log equal the oracle's step-at-a-time sums bit for bit, and
    H1 ran fewer passes than steps."""
    shapes = [(96, 320), (64, 512), (128, 200)]
    pdt = gdt
    hp_o = orc.AdamHP(lr=1e-3)
    ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], grad_dtype=TDT[gdt], param_dtype=TDT[pdt],
                     topk_ratio_ppm=100000, refresh_interval=N, accum_interval=S, adam=zf.adam_params(lr=1e-3),
                     offload=True, host_accumulate=True, cpu_update=cpu, host_stages=host_stages)
    scales = [gpu.ColScale(m, li) for li, (n, m) in enumerate(shapes)]
    Gs = [torch.empty(n, m, dtype=TDT[gdt], device="cuda") for n, m in shapes]
    Ps = [torch.empty(n, m, dtype=TDT[pdt], device="cuda") for n, m in shapes]
    for li, P in enumerate(Ps):
        gpu.fill_param(P, li)
    layers = [orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=N, accum_interval=S, hp=hp_o,
                              cpu_update=cpu) for n, m in shapes]
    Po = [np.ascontiguousarray(to_np(P)) for P in Ps]
    steps = 3 * N
    for t in range(steps):
        for li, (G, sc) in enumerate(zip(Gs, scales)):
            sc.advance_to(t)
            gpu.fill_grad(G, li, t, sc)
        Gn = [np.ascontiguousarray(to_np(G)) for G in Gs]
        ctx.step(t, Gs, Ps)
        refresh = t % N == 0
        end = (t + 1) % S == 0
        if refresh:
            ctx.sync()  # the refresh's selection drives the oracle (O10)
        for li, L in enumerate(layers):
            L.step(t, Gn[li], Po[li], idx_override=to_np(ctx.selected(li)) if refresh else None)
        if end:
            ctx.sync()
            for li, L in enumerate(layers):
                assert_bits_equal(ctx.host_accumulator(li, 0).copy(), L.acc[(t // S) % 2], f"acc t={t} l={li}")
                assert_bits_equal(ctx.host_accumulator(li, 1).copy(), L.sealed(t), f"sealed t={t} l={li}")
                assert_bits_equal(np.ascontiguousarray(to_np(Ps[li])), Po[li], f"params t={t} l={li}")
    log = ctx.window_log()
    passes, covered = ctx.host_stats()
    ctx.close()
    assert [e for (e, end, *_r) in log if end] == [t for t in range(steps) if (t + 1) % S == 0]
    assert covered == steps
    if host_stages >= 3:
        assert passes < steps, (passes, steps)


@pytest.mark.parametrize("cpu,host_stages", [(False, 8), (True, 8), (False, 16)])
def test_h1_window_batches_zen_auto(zf, orc, gpu, cpu, host_stages):
    """Zen-auto (R21) with H1 in window batches: H1 reads each staged step's K6 decision
    before forming a batch, so batches never cross a variable-length window's end; no
    zf_sync inside windows; final window log, both accumulators and the parameters equal
    the oracle's."""
    shapes, N, smax, gamma, steps = AUTO_SHAPES, 8, 8, 0.15, 24
    hp_o = orc.AdamHP(lr=1e-3)
    ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], grad_dtype=torch.bfloat16,
                     param_dtype=torch.bfloat16, topk_ratio_ppm=100000, refresh_interval=N, accum_interval=smax,
                     adam=zf.adam_params(lr=1e-3), offload=True, host_accumulate=True, cpu_update=cpu,
                     auto_gamma=gamma, host_stages=host_stages)
    scales = [gpu.ColScale(m, li) for li, (n, m) in enumerate(shapes)]
    Gs = [torch.empty(n, m, dtype=torch.bfloat16, device="cuda") for n, m in shapes]
    Ps = [torch.empty(n, m, dtype=torch.bfloat16, device="cuda") for n, m in shapes]
    for li, P in enumerate(Ps):
        gpu.fill_param(P, li)
    model = orc.OracleModel([orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=N, accum_interval=smax,
                                             hp=hp_o, cpu_update=cpu) for n, m in shapes], auto_gamma=gamma)
    Po = [np.ascontiguousarray(to_np(P)) for P in Ps]
    for t in range(steps):
        for li, (G, sc) in enumerate(zip(Gs, scales)):
            sc.advance_to(t)
            gpu.fill_grad(G, li, t, sc)
        Gn = [np.ascontiguousarray(to_np(G)) for G in Gs]
        ctx.step(t, Gs, Ps)
        ov = None
        if t % N == 0:
            ctx.sync()
            ov = [to_np(ctx.selected(li)) for li in range(len(shapes))]
        w_before = model.w
        model.step(t, Gn, Po, idx_overrides=ov)
    ctx.sync()
    ends = [e for (e, end, *_r) in ctx.window_log() if end]
    assert ends == model.ends
    for li, L in enumerate(model.layers):
        assert_bits_equal(ctx.host_accumulator(li, 0).copy(), L.acc[w_before % 2], f"acc l={li}")
        assert_bits_equal(ctx.host_accumulator(li, 1).copy(), L.acc[(model.w - 1) % 2], f"sealed l={li}")
        assert_bits_equal(np.ascontiguousarray(to_np(Ps[li])), Po[li], f"params l={li}")
    passes, covered = ctx.host_stats()
    ctx.close()
    assert covered == steps and passes < steps, (passes, covered)
    iv = model.intervals()
    assert min(iv) < smax, iv


# ------------------------------------------------------------------ randomized configurations
def _random_config(seed):
    rng = np.random.default_rng(0x5EED + seed)
    nl = int(rng.integers(1, 4))
    shapes = []
    for _ in range(nl):
        n = int(rng.choice([0, 1, 7, 33, 64, 130, 257])) if nl > 1 else int(rng.choice([1, 33, 130, 257]))
        m = int(rng.choice([33, 96, 300, 512, 777, 1025, 2048]))
        shapes.append((n, m))
    if all(n == 0 for n, _ in shapes):
        shapes[0] = (17, shapes[0][1])
    gdt = str(rng.choice(["bf16", "fp32"]))
    pdt = gdt if rng.random() < 0.7 else ("fp32" if gdt == "bf16" else "bf16")
    S = int(rng.choice([1, 2, 4]))
    N = S * int(rng.choice([1, 2]))
    ppm = int(rng.choice([2000, 10000, 100000, 250000, 1000000]))
    kw = dict(offload=bool(rng.random() < 0.8), psub=bool(rng.random() < 0.7), lr=float(rng.choice([1e-3, 1e-4])))
    if kw["offload"]:
        kw["cpu_update"] = bool(rng.random() < 0.4)
        kw["host_stages"] = int(rng.choice([0, 3, 8]))
        kw["devacc"] = bool(rng.random() < 0.25)
        if kw["cpu_update"] and rng.random() < 0.5:
            kw["cpu_async"] = True
        if rng.random() < 0.2:
            kw["side_stream"] = True
    kw["state_offload"] = bool(rng.random() < 0.15)
    if rng.random() < 0.3:
        kw["lagged"] = True
    if rng.random() < 0.3:
        kw["warmup"] = int(rng.integers(1, 3))
    if seed >= 60:   # soak-only draws (the default 60 seeds keep their configurations)
        if not kw.get("lagged") and rng.random() < 0.15:
            kw["refresh_group_mb"] = 1     # f4 (i) grouped refresh
        if rng.random() < 0.2:
            kw["poke"] = {int(rng.integers(1, 3 * N))}   # the caller rewrites p (zf_params_changed)
        if rng.random() < 0.15:            # one larger, ragged layer
            shapes.append((int(rng.integers(200, 520)), int(rng.integers(2000, 4100))))
    return shapes, gdt, pdt, ppm, N, S, kw


# ZF_RANDOM_SEEDS widens the sweep (a soak run; the default suite runs the first 60)
@pytest.mark.parametrize("seed", range(int(os.environ.get("ZF_RANDOM_SEEDS", "60"))))
def test_step_random_configurations(zf, orc, gpu, seed):
    """Seeded random mixes of the context's options (shapes incl. rows-less and ragged layers,
    fp32 / bf16 / mixed dtypes, ratios 0.2%..100%, N and S, offload, f1, host staging slots,
    K7 device accumulation, state swap-out, overlapped f1, a caller side stream, param_subset,
    lagged selection, warm-up), each
    run for three refresh periods: selection,
    moments, step counts, parameters, compact blocks and accumulators bit-exact."""
    shapes, gdt, pdt, ppm, N, S, kw = _random_config(seed)
    steps = kw.get("warmup", 0) + 3 * N + 1
    _run_stateful(zf, orc, gpu, shapes, gdt, pdt, ppm, N, S, steps, **kw)
