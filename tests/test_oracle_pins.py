"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every test here checks the oracle against something OTHER than itself: a
worked example printed in the reference (tests/golden/, each cited), a closed
form, an invariant, a brute-force evaluation on tiny inputs written
independently (different loop order / definition), or a library routine
(torch.optim.AdamW, torch's bf16 cast) for a special case the method reduces
to.  Each is chosen so a plausible slip in the oracle (a dropped term, a
transposed operand, a wrong index or sign) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _bf16(x):
    """bf16 bit patterns via torch's own RNE cast (a library routine)."""
    t = torch.tensor(np.asarray(x, np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


# ------------------------------------------------------------------ bf16 RNE
def test_bf16_round_matches_torch(orc):
    rng = np.random.default_rng(1)
    xs = np.concatenate([rng.standard_normal(2000).astype(np.float32) * 10.0 ** rng.integers(-8, 8, 2000),
                         np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -(1.0 + 2 ** -8), 0.0, -0.0], np.float32)])
    want = orc.bf16_bits_to_f32(_bf16(xs))
    got = np.array([orc.bf16_round(float(x)) for x in xs], np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_bf16_nan_with_low_payload_stays_nan(orc):
    """A NaN whose payload sits only in the 16 dropped bits must stay a NaN in bf16 (torch's
    cast gives a NaN too), not collapse to the infinity that plain truncation of 0x7f800001
    gives -- the non-finite check (R15) relies on it.  Sign and payload are not compared:
    torch returns one canonical NaN."""
    for bits in (0x7F800001, 0xFF800001, 0x7F80FFFF, 0x7FC00000):
        x = np.array([bits], np.uint32).view(np.float32)
        want = orc.bf16_bits_to_f32(_bf16(x))
        got = orc.to_bf16(x)
        assert np.isnan(orc.bf16_bits_to_f32(got)).all() and np.isnan(want).all(), hex(bits)


# ------------------------------------------------------------------ O2  k
def test_k_closed_form_table(orc):
    for m, k10, k1 in _golden("k_table.json")["rows"]:
        assert orc.k_for(m, 100000) == k10, m
        assert orc.k_for(m, 10000) == k1, m


def test_k_integer_ceil_edge(orc):
    # 100 * 0.07 = 7.000000000000001 in binary fp -> a float ceil gives 8; ceil(7) = 7.
    assert orc.k_for(100, 70000) == 7
    assert orc.k_for(1, 1) == 1            # k >= 1
    assert orc.k_for(37, 1000000) == 37    # ratio 1 -> all columns
    for m in range(1, 300):
        for ppm in (1, 9999, 10000, 100000, 333333, 999999):
            assert orc.k_for(m, ppm) == max(1, -(-m * ppm // 1000000))


# ------------------------------------------------------------------ O1  norms
def test_norms_worked_examples(orc):
    for ex in _golden("worked_examples.json")["column_norms"]:
        G = np.array(ex["G"], np.float32)
        assert np.array_equal(orc.column_norms(G), np.array(ex["norms"], np.float32)), ex["source"]


def test_norms_sharded_worked_example(orc):
    ex = _golden("worked_examples.json")["gather_column_norms"][0]
    parts = [orc.column_norms_f64(np.array(s, np.float32)) for s in ex["shards"]]
    assert np.array_equal(sum(parts), np.array(ex["norms"])), ex["source"]


def test_norms_integer_closed_form(orc):
    # G[i][j] = i + j (exact in bf16 for these sizes): sum_i (i+j)^2 =
    #   n(n-1)(2n-1)/6 + j n(n-1) + n j^2, an exact integer < 2^24.
    n, m = 40, 24
    G = np.add.outer(np.arange(n), np.arange(m)).astype(np.float32)
    for dt, arr in (("fp32", G), ("bf16", _bf16(G))):
        got = orc.column_norms(arr)
        j = np.arange(m)
        want = n * (n - 1) * (2 * n - 1) // 6 + j * n * (n - 1) + n * j * j
        assert np.array_equal(got, want.astype(np.float32)), dt


def test_norms_frobenius_invariant(orc):
    rng = np.random.default_rng(7)
    G = (rng.standard_normal((300, 257)) * np.exp(rng.standard_normal(257) * 2)).astype(np.float32)
    cn = orc.column_norms_f64(G)
    frob = math.fsum(float(x) * float(x) for x in G.ravel())          # row-major, compensated
    assert abs(math.fsum(cn) - frob) <= 1e-12 * frob
    assert np.allclose(orc.column_norms(G), cn.astype(np.float32), rtol=0, atol=0)


def test_norms_brute_force_64(orc):
    rng = np.random.default_rng(3)
    G = rng.standard_normal((64, 64)).astype(np.float32)
    got = orc.column_norms(G)
    for j in range(64):                     # independent loop: rows outer, via python floats
        s = math.fsum(float(G[i, j]) ** 2 for i in range(64))
        assert abs(float(got[j]) - s) <= 2 ** -23 * s


def test_norms_shard_sum(orc):
    rng = np.random.default_rng(4)
    G = rng.standard_normal((103, 50)).astype(np.float32)
    whole = orc.column_norms_f64(G)
    for world in (2, 3, 8):
        parts = [orc.column_norms_f64(G[slice(*orc.shard_rows(103, world, r))]) for r in range(world)]
        assert np.allclose(sum(parts), whole, rtol=1e-12, atol=0)


def test_strided_rows_read_only_the_first_m_columns(orc):
    """Row i of G / p starts at i*ld (SURVEY §8(b) layout, ld >= m): the C oracle called on a
    padded buffer gives the norms (against numpy's float64 sum of squares), the compaction
    and the AdamW results of the dense [n, m] matrix, and never touches the padding."""
    import ctypes
    rng = np.random.default_rng(7)
    n, m, ld = 9, 13, 21
    Gp = np.full((n, ld), 1.0e3, np.float32)
    Gp[:, :m] = rng.standard_normal((n, m)).astype(np.float32)
    G = np.ascontiguousarray(Gp[:, :m])
    L = orc.lib()
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    norms = np.empty(m, np.float32)
    assert L.oracle_column_norms(vp(Gp), orc.F32, n, m, ld, vp(norms)) == 0
    want = (G.astype(np.float64) ** 2).sum(axis=0).astype(np.float32)
    assert np.array_equal(norms, want)
    idx = np.array([1, 4, 12], np.int32)
    out = np.empty((n, m - 3), np.float32)
    L.oracle_compact(vp(Gp), orc.F32, n, m, ld, vp(idx), 3, vp(out))
    assert np.array_equal(out, np.delete(G, idx, axis=1))
    Pp = np.full((n, ld), -7.0, np.float32)
    Pp[:, :m] = rng.standard_normal((n, m)).astype(np.float32)
    P = np.ascontiguousarray(Pp[:, :m])
    M1, V1, s1 = np.zeros((n, 3), np.float32), np.zeros((n, 3), np.float32), np.zeros(3, np.int32)
    M2, V2, s2 = M1.copy(), V1.copy(), s1.copy()
    L.oracle_selective_adamw(vp(Pp), orc.F32, ld, vp(Gp), orc.F32, ld, n, vp(idx), 3, vp(M1), vp(V1), vp(s1),
                             1e-3, 0.9, 0.999, 1e-8, 0.0, 1)
    orc.selective_adamw(P, G, idx, M2, V2, s2, orc.AdamHP())
    assert np.array_equal(Pp[:, :m], P) and np.array_equal(M1, M2) and np.array_equal(V1, V2)
    assert np.all(Pp[:, m:] == -7.0)


def test_norms_reject_nonfinite(orc):
    G = np.ones((4, 4), np.float32)
    G[2, 1] = np.nan
    with pytest.raises(FloatingPointError):
        orc.column_norms(G)


def test_topk_rejects_nonfinite_norms(orc):
    """SPEC S:44 / S:108 reject non-finite input (reading R15): a NaN or infinite norm is an
    error, not a column that wins (inf) or loses (NaN) the ranking."""
    for bad in (np.nan, np.inf):
        norms = np.array([1.0, bad, 0.5, 2.0], np.float32)
        with pytest.raises(FloatingPointError):
            orc.topk(norms, 2)


# ------------------------------------------------------------------ O3  top-k
def test_topk_worked_examples(orc):
    for ex in _golden("worked_examples.json")["select_channels"]:
        norms = np.array(ex["norms"], np.float32)
        k = orc.k_for(len(norms), ex["ratio_ppm"])
        assert orc.topk(norms, k).tolist() == ex["idx"], ex["source"]


def _rank_count_select(norms, k):
    # independent definition: rank_j = #{i: N_i > N_j or (N_i == N_j and i < j)}; selected iff rank_j < k
    m = len(norms)
    sel = []
    for j in range(m):
        r = sum(1 for i in range(m) if norms[i] > norms[j] or (norms[i] == norms[j] and i < j))
        if r < k:
            sel.append(j)
    return sel


def test_topk_brute_force_with_ties(orc):
    rng = np.random.default_rng(11)
    for trial in range(200):
        m = int(rng.integers(1, 65))
        norms = rng.integers(0, 6, m).astype(np.float32) * 0.25     # many exact ties
        k = int(rng.integers(1, m + 1))
        assert orc.topk(norms, k).tolist() == _rank_count_select(norms.tolist(), k), (trial, m, k)


def test_topk_permutation_equivariance(orc):
    rng = np.random.default_rng(12)
    norms = rng.standard_normal(500).astype(np.float32) ** 2       # distinct values
    k = 50
    base = set(orc.topk(norms, k).tolist())
    perm = rng.permutation(500)
    got = set(perm[j] for j in orc.topk(norms[perm], k).tolist())
    assert got == base


def test_topk_concentrated_columns(orc):
    # nonzeros confined to c <= k columns -> all of them are selected
    rng = np.random.default_rng(13)
    G = np.zeros((30, 100), np.float32)
    cols = rng.choice(100, 7, replace=False)
    G[:, cols] = rng.standard_normal((30, 7)).astype(np.float32) + 3.0
    idx = orc.topk(orc.column_norms(G), 10)
    assert set(cols.tolist()) <= set(idx.tolist())
    assert list(idx) == sorted(idx)


# ------------------------------------------------------------------ O4  map
def test_column_map_definition(orc):
    rng = np.random.default_rng(5)
    m = 97
    idx = np.sort(rng.choice(m, 13, replace=False)).astype(np.int32)
    slot, upos = orc.column_map(idx, m)
    unsel = [j for j in range(m) if j not in set(idx.tolist())]
    for j in range(m):
        if j in set(idx.tolist()):
            assert slot[j] == idx.tolist().index(j) and upos[j] == -1
        else:
            assert slot[j] == -1 and upos[j] == unsel.index(j)


# ------------------------------------------------------------------ O7  compaction
def test_compact_worked_example(orc):
    ex = _golden("worked_examples.json")["mask_from_channels"][0]
    G = np.arange(ex["rows"] * ex["cols"], dtype=np.float32).reshape(ex["rows"], ex["cols"])
    out = orc.compact(G, np.array(ex["idx"], np.int32))
    assert out.shape == (ex["rows"], ex["cols"] - len(ex["idx"]))
    assert np.array_equal(out, G[:, ex["unselected_columns"]]), ex["source"]
    assert ex["rows"] * len(ex["idx"]) == ex["n_selected_elements"]


def test_compact_partition_identity(orc):
    # O9: |idx| + |unsel| = m, disjoint, and every row rebuilds bit for bit
    rng = np.random.default_rng(6)
    for dt in ("fp32", "bf16"):
        n, m = 37, 211
        Gf = rng.standard_normal((n, m)).astype(np.float32)
        G = Gf if dt == "fp32" else _bf16(Gf)
        idx = orc.topk(orc.column_norms(G), orc.k_for(m, 100000))
        out = orc.compact(G, idx)
        slot, upos = orc.column_map(idx, m)
        R = np.empty_like(G)
        for j in range(m):
            R[:, j] = G[:, idx[slot[j]]] if slot[j] >= 0 else out[:, upos[j]]
        assert np.array_equal(R.view(np.uint8), G.view(np.uint8))
        assert len(set(idx.tolist())) == len(idx) and out.shape[1] + len(idx) == m


def test_compact_all_selected_is_empty(orc):
    G = np.ones((5, 8), np.float32)
    assert orc.compact(G, np.arange(8, dtype=np.int32)).shape == (5, 0)


def test_compact_shards_concatenate(orc):
    rng = np.random.default_rng(8)
    G = _bf16(rng.standard_normal((21, 40)))
    idx = np.array([0, 5, 6, 39], np.int32)
    whole = orc.compact(G, idx)
    parts = [orc.compact(np.ascontiguousarray(G[slice(*orc.shard_rows(21, 4, r))]), idx) for r in range(4)]
    assert np.array_equal(np.concatenate(parts), whole)


def test_shard_rows_worked_examples(orc):
    for ex in _golden("worked_examples.json")["shard_matrix"]:
        rows = [b - a for a, b in (orc.shard_rows(ex["n"], ex["world"], r) for r in range(ex["world"]))]
        assert rows == ex["rows"], ex["source"]


def test_byte_accounting_worked_example():
    ex = _golden("worked_examples.json")["byte_accounting"][0]
    assert 4096 * 4096 * 2 == ex["full_bytes"] and 4096 * 4 == ex["proxy_bytes"]


# ------------------------------------------------------------------ O6  AdamW
def _adam_state(n, k):
    return np.zeros((n, k), np.float32), np.zeros((n, k), np.float32), np.zeros(k, np.int32)


def test_adam_step1_closed_form(orc):
    # from zero state, m_hat = g and v_hat = g^2, so p1 = p0 - lr * g / (|g| + eps)
    rng = np.random.default_rng(20)
    n, m = 16, 12
    G = (rng.standard_normal((n, m)) * 1e-2).astype(np.float32)
    P = rng.standard_normal((n, m)).astype(np.float32)
    P0 = P.copy()
    idx = np.array([1, 4, 5, 11], np.int32)
    M, V, st = _adam_state(n, 4)
    hp = orc.AdamHP(lr=1e-3)
    orc.selective_adamw(P, G, idx, M, V, st, hp)
    g = G[:, idx].astype(np.float64)
    want = P0[:, idx].astype(np.float64) - 1e-3 * g / (np.abs(g) + 1e-8)
    assert np.allclose(P[:, idx], want, rtol=1e-6, atol=0)
    other = np.setdiff1d(np.arange(m), idx)
    assert np.array_equal(P[:, other], P0[:, other])            # unselected untouched
    assert st.tolist() == [1, 1, 1, 1]
    assert np.allclose(M, 0.1 * G[:, idx], rtol=1e-6) and np.allclose(V, 0.001 * G[:, idx] ** 2, rtol=1e-5)


def test_adam_constant_gradient_closed_form(orc):
    # constant g: m_hat_t = g and v_hat_t = g^2 for every t, so each step moves p by -lr*g/(|g|+eps)
    n = 8
    G = np.linspace(-0.05, 0.05, n * 3, dtype=np.float32).reshape(n, 3)
    G[G == 0] = 0.01
    P = np.zeros((n, 3), np.float32)
    idx = np.array([0, 1, 2], np.int32)
    M, V, st = _adam_state(n, 3)
    hp = orc.AdamHP(lr=1e-2)
    for t in range(1, 9):
        orc.selective_adamw(P, G, idx, M, V, st, hp)
        g = G.astype(np.float64)
        assert np.allclose(P, -t * 1e-2 * g / (np.abs(g) + 1e-8), rtol=2e-6, atol=0), t


@pytest.mark.parametrize("wd,decoupled", [(0.0, 1), (0.01, 1), (0.01, 0)])
def test_adam_all_selected_equals_torch(orc, wd, decoupled):
    # k = m: every column selected from t=1 -> the plain optimizer (O6 library case)
    rng = np.random.default_rng(21)
    n, m = 24, 10
    P = rng.standard_normal((n, m)).astype(np.float32)
    tp = torch.nn.Parameter(torch.tensor(P.copy()))
    cls = torch.optim.AdamW if decoupled else torch.optim.Adam
    opt = cls([tp], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=wd, foreach=False)
    M, V, st = _adam_state(n, m)
    hp = orc.AdamHP(lr=1e-3, weight_decay=wd, decoupled=decoupled)
    idx = np.arange(m, dtype=np.int32)
    for t in range(6):
        G = (rng.standard_normal((n, m)) * 10.0 ** rng.integers(-4, 0)).astype(np.float32)
        orc.selective_adamw(P, G, idx, M, V, st, hp)
        tp.grad = torch.tensor(G)
        opt.step()
        ref = tp.detach().numpy()
        assert np.allclose(P, ref, rtol=1e-6, atol=1e-9), t
        state = opt.state[tp]
        # torch forms m with lerp (a few ulps of the terms apart from b1*m + (1-b1)*g),
        # so moments are compared norm-wise: |diff| <= 1e-6 * max|ref|
        for mine, ref_t in ((M, state["exp_avg"]), (V, state["exp_avg_sq"])):
            ref_m = ref_t.numpy()
            assert np.max(np.abs(mine - ref_m)) <= 1e-6 * np.max(np.abs(ref_m))


def test_adam_bf16_param_within_one_ulp_of_torch_fp32_then_round(orc):
    rng = np.random.default_rng(22)
    n, m = 32, 16
    Pf = rng.standard_normal((n, m)).astype(np.float32) * 0.02
    Pb = _bf16(Pf)
    Gb = _bf16(rng.standard_normal((n, m)) * 1e-3)
    idx = np.arange(m, dtype=np.int32)
    M, V, st = _adam_state(n, m)
    orc.selective_adamw(Pb, Gb, idx, M, V, st, orc.AdamHP(lr=1e-3))
    tp = torch.nn.Parameter(torch.tensor(orc.bf16_bits_to_f32(Pb.copy()) * 0 + orc.bf16_bits_to_f32(_bf16(Pf))))
    opt = torch.optim.AdamW([tp], lr=1e-3, weight_decay=0.0, foreach=False)
    tp.grad = torch.tensor(orc.bf16_bits_to_f32(Gb))
    opt.step()
    ref = _bf16(tp.detach().numpy()).astype(np.int32)
    assert np.max(np.abs(Pb.astype(np.int32) - ref)) <= 1       # within 1 bf16 ulp


def test_adam_per_slot_step_counts(orc):
    # slots with different ages use their own bias correction: a slot at step 0 moves by ~lr
    n = 4
    G = np.full((n, 2), 0.5, np.float32)
    P = np.zeros((n, 2), np.float32)
    idx = np.array([0, 1], np.int32)
    M = np.zeros((n, 2), np.float32)
    V = np.zeros((n, 2), np.float32)
    st = np.array([0, 100], np.int32)
    M[:, 1] = 0.5
    V[:, 1] = 0.25
    orc.selective_adamw(P, G, idx, M, V, st, orc.AdamHP(lr=1e-3))
    assert st.tolist() == [1, 101]
    b1, b2 = 0.9, 0.999
    # slot 1: m stays 0.5 and v stays 0.25; bias corrections at t=101
    want1 = -1e-3 / (1 - b1 ** 101) * 0.5 / (math.sqrt(0.25) / math.sqrt(1 - b2 ** 101) + 1e-8)
    assert np.allclose(P[:, 0], -1e-3 * 0.5 / (0.5 + 1e-8), rtol=1e-6)
    assert np.allclose(P[:, 1], want1, rtol=1e-6)


# ------------------------------------------------------------------ O5  remap (reading R7)
def test_remap_persistent_column_follows_plain_adamw(orc):
    """Invariant of reading R7: a column selected on every step follows plain AdamW
    exactly, whatever the other selected columns do across refreshes."""
    rng = np.random.default_rng(30)
    n, m = 6, 20
    Pcol = rng.standard_normal(n).astype(np.float32)
    tp = torch.nn.Parameter(torch.tensor(Pcol.copy()))
    opt = torch.optim.AdamW([tp], lr=1e-3, weight_decay=0.0, foreach=False)
    layer = orc.OracleLayer(n=n, m=m, ratio_ppm=150000, refresh_interval=2, accum_interval=2)
    P = rng.standard_normal((n, m)).astype(np.float32)
    P[:, 7] = Pcol
    for t in range(10):
        G = (rng.standard_normal((n, m)) * 0.01).astype(np.float32)
        G[:, 7] = (rng.standard_normal(n) + 50.0).astype(np.float32)    # column 7 always the largest
        layer.step(t, G, P)
        assert 7 in layer.idx.tolist()
        tp.grad = torch.tensor(G[:, 7].copy())
        opt.step()
        assert np.allclose(P[:, 7], tp.detach().numpy(), rtol=1e-6, atol=1e-9), t


def test_remap_no_refresh_equals_constant_selection(orc):
    # N = infinity (refresh only at t=0) vs N = 1 with a selection that never changes
    rng = np.random.default_rng(31)
    n, m = 5, 30
    Gs = [(rng.standard_normal((n, m)) * 0.01).astype(np.float32) for _ in range(6)]
    for G in Gs:
        G[:, [2, 9, 17]] += 10.0
    P0 = rng.standard_normal((n, m)).astype(np.float32)
    a = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=1000, accum_interval=1)
    b = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=1, accum_interval=1)
    Pa, Pb = P0.copy(), P0.copy()
    for t, G in enumerate(Gs):
        a.step(t, G, Pa)
        b.step(t, G, Pb)
        assert a.idx.tolist() == b.idx.tolist() == [2, 9, 17]
    assert np.array_equal(Pa, Pb) and np.array_equal(a.M, b.M) and np.array_equal(a.V, b.V)


def test_remap_retained_entering_leaving(orc):
    # reading R7 worked by hand (parity unpinned beyond internal consistency: paper silent)
    n = 2
    idx_old = np.array([1, 3], np.int32)
    M_old = np.array([[1, 2], [3, 4]], np.float32)
    V_old = M_old * 10
    st_old = np.array([5, 7], np.int32)
    M, V, st = orc.remap(n, idx_old, M_old, V_old, st_old, np.array([3, 5], np.int32))
    assert M.tolist() == [[2, 0], [4, 0]] and V.tolist() == [[20, 0], [40, 0]] and st.tolist() == [7, 0]


def test_remap_entering_column_restarts_from_the_step1_closed_form(orc):
    """R7 on whole steps, against closed forms: a column that enters the selection at a
    refresh starts AdamW from zero moments and step count, so its first GPU update is the
    bias-corrected step-1 move p - lr*g/(|g|+eps); a column that leaves and re-enters later
    restarts the same way; a retained column continues its sequence (step 2 from a constant
    g is again -lr*g/(|g|+eps), m_hat = g, v_hat = g^2)."""
    n, m, lr, eps = 3, 10, 1e-3, 1e-8
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=2, accum_interval=2, hp=orc.AdamHP(lr=lr))
    P = np.zeros((n, m), np.float32)

    def G_top(col, g=0.5):
        G = np.full((n, m), 0.01, np.float32)
        G[:, col] = g
        return G

    for t, top in enumerate([2, 2, 7, 7, 2, 2]):   # column 2, then 7 (entering), then 2 again (re-entering)
        before = P.copy()
        L.step(t, G_top(top), P)
        assert L.idx.tolist() == [top]
        d = P[:, top] - before[:, top]
        want = -lr * 0.5 / (0.5 + eps)
        assert np.allclose(d, want, rtol=1e-6), (t, d, want)    # step 1 (entering) and step 2 (retained)
        assert L.steps.tolist() == [1 + t % 2]                   # the step count restarts at each entry


# ------------------------------------------------------------------ O8  accumulation
def test_accumulate_constant_dyadic_stream(orc):
    # dyadic values: fp32 sums are exact, so after S steps acc = S * g exactly
    g = (np.arange(-50, 50, dtype=np.float32) * 2.0 ** -10).reshape(4, 25)
    for dt, stage in (("fp32", g), ("bf16", _bf16(g))):
        acc = np.zeros_like(g)
        for _ in range(4):
            orc.accumulate(acc, stage)
        assert np.array_equal(acc, 4 * g), dt


def test_window_double_buffer(orc):
    # S=2: windows [0,2), [2,4) alternate buffers; a buffer holds exactly its window's steps
    n, m = 3, 10
    layer = orc.OracleLayer(n=n, m=m, ratio_ppm=200000, refresh_interval=2, accum_interval=2)
    P = np.zeros((n, m), np.float32)
    outs = []
    for t in range(4):
        G = np.full((n, m), float(t + 1), np.float32) * np.arange(1, m + 1, dtype=np.float32)
        outs.append(layer.step(t, G, P).copy())
    assert np.array_equal(layer.acc[0], outs[0] + outs[1])
    assert np.array_equal(layer.acc[1], outs[2] + outs[3])
    assert layer.sealed(3) is layer.acc[1] and layer.sealed(1) is layer.acc[0]
    assert layer.sealed(2) is layer.acc[0]      # mid-window: the last SEALED window, not the active one
    assert layer.sealed(0) is None              # nothing sealed before the first window ends


def test_accumulate_S1_is_the_compact_gradient(orc):
    rng = np.random.default_rng(40)
    layer = orc.OracleLayer(n=4, m=12, ratio_ppm=250000, refresh_interval=1, accum_interval=1)
    P = np.zeros((4, 12), np.float32)
    G = rng.standard_normal((4, 12)).astype(np.float32)
    out = layer.step(0, G, P)
    unsel = [j for j in range(12) if j not in set(layer.idx.tolist())]
    assert np.array_equal(layer.acc[0], G[:, unsel]) and np.array_equal(out, G[:, unsel])


def test_step_all_important_equals_plain_optimizer(orc):
    # mask = all-important -> theta^(c) empty; trajectory = plain AdamW
    rng = np.random.default_rng(41)
    n, m = 7, 9
    P = rng.standard_normal((n, m)).astype(np.float32)
    tp = torch.nn.Parameter(torch.tensor(P.copy()))
    opt = torch.optim.AdamW([tp], lr=1e-3, weight_decay=0.0, foreach=False)
    layer = orc.OracleLayer(n=n, m=m, ratio_ppm=1000000, refresh_interval=4, accum_interval=4)
    for t in range(8):
        G = rng.standard_normal((n, m)).astype(np.float32)
        out = layer.step(t, G, P)
        assert out.shape == (n, 0)
        tp.grad = torch.tensor(G)
        opt.step()
    assert np.allclose(P, tp.detach().numpy(), rtol=1e-6, atol=1e-9)


# ------------------------------------------------------------------ f1: deferred CPU AdamW (reading R18)
def test_f1_S1_constant_selection_is_plain_adamw(orc):
    """S = N = 1 with a selection that never changes: the GPU side (selected columns) and the
    deferred CPU side (the rest, flushed every step with the 1-step average) together are
    plain AdamW on the whole matrix (SPEC S:268 degenerate interval; P:519-531 with S=1)."""
    rng = np.random.default_rng(50)
    n, m = 6, 20
    P = (rng.standard_normal((n, m)) * 0.1).astype(np.float32)
    tp = torch.nn.Parameter(torch.tensor(P.copy()))
    opt = torch.optim.AdamW([tp], lr=1e-3, weight_decay=0.0, foreach=False)
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=150000, refresh_interval=1, accum_interval=1, cpu_update=True)
    for t in range(8):
        G = (rng.standard_normal((n, m)) * 0.01).astype(np.float32)
        G[:, [3, 11, 17]] += 5.0                       # these three columns always selected
        L.step(t, G, P)
        assert L.idx.tolist() == [3, 11, 17]
        tp.grad = torch.tensor(G)
        opt.step()
        assert np.allclose(P, tp.detach().numpy(), rtol=1e-6, atol=1e-9), t


def test_f1_window_average_closed_form(orc):
    """S = 2, constant gradient: an unselected column moves only at window ends, each time by
    one bias-corrected AdamW step with the window average (= g): -lr*g/(|g|+eps) at its
    first flush (theta^(c) -= alpha * (1/S) * sum over the window)."""
    n, m = 4, 10
    G = np.full((n, m), 0.25, np.float32)
    G[:, 0] = 9.0                                      # column 0 selected (k = 1)
    P = np.zeros((n, m), np.float32)
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=2, accum_interval=2, cpu_update=True)
    L.step(0, G, P)
    assert np.all(P[:, 1:] == 0.0)                     # mid-window: CPU columns unchanged
    L.step(1, G, P)
    want = -1e-3 * 0.25 / (0.25 + 1e-8)
    assert np.allclose(P[:, 1:], want, rtol=1e-6)
    assert L.th[1:].tolist() == [1] * (m - 1) and L.th[0] == 0
    L.step(2, G, P)
    assert np.allclose(P[:, 1:], want, rtol=1e-6)      # unchanged until the window ends
    L.step(3, G, P)
    assert np.allclose(P[:, 1:], 2 * want, rtol=1e-5)  # constant g: m_hat = g, v_hat = g^2 again


def test_f1_migration_takes_current_value(orc):
    """A column leaving the GPU-updated set takes the parameter's current value as its
    fp32 master, with zero host moments and step count (reading R18)."""
    n, m = 3, 8
    P = np.zeros((n, m), np.float32)
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=125000, refresh_interval=2, accum_interval=2, cpu_update=True)
    G = np.full((n, m), 0.5, np.float32)
    G[:, 2] = 7.0                                      # window 0: column 2 on the GPU
    L.step(0, G, P)
    L.step(1, G, P)
    p2 = P[:, 2].copy()
    assert np.all(p2 != 0.0) and L.th[2] == 0
    G2 = np.full((n, m), 0.5, np.float32)
    G2[:, 5] = 7.0                                     # window 1: column 5 on the GPU, 2 back on the CPU
    L.step(2, G2, P)
    assert np.array_equal(L.master[:, 2], p2) and L.th[2] == 0 and np.all(L.Mh[:, 2] == 0)


def test_f1_reentering_column_restarts_from_the_step1_closed_form(orc):
    """Reading R18 on whole windows: column 5 is CPU-updated in window 0 (g = +0.25), moves to
    the GPU in window 1, and re-enters the CPU set in window 2 with g = -0.25.  It re-enters
    with zero host moments and step count, so its window-2 flush is the bias-corrected step-1
    move -lr*g/(|g|+eps) = +lr (to 4e-8), and its host step count is 1.  Keeping window 0's
    moments or count would give a different move (+0.05 lr, +0.07 lr or +0.74 lr)."""
    n, m, lr = 3, 8, 1e-3
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=125000, refresh_interval=2, accum_interval=2, cpu_update=True,
                        hp=orc.AdamHP(lr=lr))
    P = np.zeros((n, m), np.float32)

    def G(spike, g5):
        x = np.full((n, m), 0.25, np.float32)
        x[:, 5] = g5
        x[:, spike] = 7.0
        return x

    for t, (spike, g5) in enumerate([(2, 0.25), (2, 0.25), (5, 0.0), (5, 0.0)]):
        L.step(t, G(spike, g5), P)
    assert L.idx.tolist() == [5]
    before = P[:, 5].copy()
    L.step(4, G(2, -0.25), P)
    assert np.array_equal(P[:, 5], before)              # mid-window: unchanged
    L.step(5, G(2, -0.25), P)
    assert L.idx.tolist() == [2] and L.th[5] == 1
    assert np.allclose(P[:, 5] - before, _step1_move(-0.25, lr=lr), rtol=1e-5, atol=0)
    assert np.array_equal(L.Mh[:, 5], np.full(n, np.float32(0.1) * np.float32(-0.25), np.float32))


def test_f1_flush_leaves_the_selected_columns_alone_bf16(orc):
    """bf16 parameters: a window flush writes only theta^(c) (the unselected columns); the
    selected column keeps the GPU-side AdamW result (two step-1-shaped moves of -lr*g/(|g|+eps)
    on a constant g, each rounded to bf16), not a value from the host master."""
    n, m, lr = 3, 8, 2.0 ** -7
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=125000, refresh_interval=2, accum_interval=2, cpu_update=True,
                        hp=orc.AdamHP(lr=lr))
    P = _bf16(np.full((n, m), 0.5, np.float32))
    G = np.full((n, m), 0.25, np.float32)
    G[:, 3] = 4.0
    L.step(0, G, P)
    L.step(1, G, P)
    assert L.idx.tolist() == [3]
    sel = orc.bf16_bits_to_f32(P[:, 3])
    want = orc.bf16_round(orc.bf16_round(0.5 + _step1_move(4.0, lr=lr)) + _step1_move(4.0, lr=lr))
    assert np.all(sel == np.float32(want)) and want < 0.5
    cpu = orc.bf16_bits_to_f32(P[:, [0, 1, 2, 4, 5, 6, 7]])
    assert np.all(cpu == np.float32(orc.bf16_round(0.5 + _step1_move(0.25, lr=lr))))


# ------------------------------------------------------------------ f2: warm-up (reading R20)
def test_f2_warmup_is_plain_adamw_on_the_whole_matrix(orc):
    """t < tau: synchronous AdamW on every column = torch.optim.AdamW on the
    full matrix; nothing is offloaded."""
    rng = np.random.default_rng(60)
    n, m = 5, 12
    P = (rng.standard_normal((n, m)) * 0.1).astype(np.float32)
    tp = torch.nn.Parameter(torch.tensor(P.copy()))
    opt = torch.optim.AdamW([tp], lr=1e-3, weight_decay=0.0, foreach=False)
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=250000, refresh_interval=2, accum_interval=2, warmup=5)
    for t in range(5):
        G = rng.standard_normal((n, m)).astype(np.float32)
        out = L.step(t, G, P)
        assert out.shape == (n, 0) and L.acc is None
        tp.grad = torch.tensor(G)
        opt.step()
        assert np.allclose(P, tp.detach().numpy(), rtol=1e-6, atol=1e-9), t


def test_f2_warmup_zero_is_the_plain_schedule(orc):
    rng = np.random.default_rng(61)
    n, m = 4, 16
    P0 = rng.standard_normal((n, m)).astype(np.float32)
    A = orc.OracleLayer(n=n, m=m, ratio_ppm=200000, refresh_interval=2, accum_interval=2, warmup=0)
    B = orc.OracleLayer(n=n, m=m, ratio_ppm=200000, refresh_interval=2, accum_interval=2)
    PA, PB = P0.copy(), P0.copy()
    for t in range(5):
        G = rng.standard_normal((n, m)).astype(np.float32)
        assert np.array_equal(A.step(t, G, PA), B.step(t, G, PB))
    assert np.array_equal(PA, PB) and np.array_equal(A.M, B.M)


def test_f2_column_selected_at_tau_continues_its_adamw_sequence(orc):
    """R20 with R7: a column that is selected at the first regular refresh (step tau) keeps
    the moments and step count it built during warm-up, so a column selected from step tau
    on follows uninterrupted AdamW from step 0 (compare with torch on that column)."""
    rng = np.random.default_rng(62)
    n, m, tau = 3, 10, 3
    P = (rng.standard_normal((n, m)) * 0.1).astype(np.float32)
    tp = torch.nn.Parameter(torch.tensor(P[:, [4]].copy()))
    opt = torch.optim.AdamW([tp], lr=1e-3, weight_decay=0.0, foreach=False)
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=2, accum_interval=2, warmup=tau)
    for t in range(tau + 4):
        G = (rng.standard_normal((n, m)) * 0.01).astype(np.float32)
        G[:, 4] += 3.0                                   # column 4 is the top column after warm-up
        L.step(t, G, P)
        if t >= tau:
            assert L.idx.tolist() == [4]
        tp.grad = torch.tensor(G[:, [4]])
        opt.step()
        assert np.allclose(P[:, [4]], tp.detach().numpy(), rtol=1e-6, atol=1e-9), t
    assert L.steps.tolist() == [tau + 4]               # one uninterrupted step count


# ------------------------------------------------------------------ f2: Zen-auto (reading R21)
def _auto_model(orc, n, m, ppm, N, smax, gamma, cpu_update=False, layers=1, warmup=0):
    Ls = [orc.OracleLayer(n=n, m=m, ratio_ppm=ppm, refresh_interval=N, accum_interval=smax,
                          cpu_update=cpu_update, warmup=warmup) for _ in range(layers)]
    return orc.OracleModel(Ls, auto_gamma=gamma)


def _two_level(n, m, k, hi, lo):
    """Constant stream: k important columns of value hi, the rest lo (per-channel L2 norm
    ratio lo/hi exactly, every step)."""
    G = np.full((n, m), lo, np.float32)
    G[:, :k] = hi
    return G


def test_zen_auto_spec_worked_example(orc):
    """per-channel norm of the unimportant part = 0.25 x the important part,
    constant stream, gamma = 1 -> the CPU-side update triggers at the 4th step of every
    window (the accumulated unimportant norm reaches 4 x 0.25 = 1 x important)."""
    ex = _golden("worked_examples.json")["zen_auto"][0]
    n, m = 16, 64
    M = _auto_model(orc, n, m, 100000, N=16, smax=16, gamma=ex["gamma"])
    k = M.layers[0].k
    G = _two_level(n, m, k, 1.0, ex["ratio"])
    P = np.zeros((n, m), np.float32)
    for t in range(16):
        M.step(t, [G], [P])
    assert M.intervals() == [ex["trigger_step"]] * 4
    assert M.ends == [3, 7, 11, 15]


def test_zen_auto_threshold_worked_example(orc):
    """gamma = 1, accumulated 0.5 vs important 0.6 -> no flush; the comparison
    is >= (0.6 accumulated flushes)."""
    ex = _golden("worked_examples.json")["zen_auto"][1]
    z = orc.ZenAuto(ex["gamma"], 100)
    assert z.decide(0.6, 1, ex["accumulated"], 1, False) is ex["flush"]
    z = orc.ZenAuto(ex["gamma"], 100)
    assert z.decide(0.6, 1, 0.6, 1, False) is True


@pytest.mark.parametrize("lo,gamma,want", [(0.25, 1.0, 4), (0.5, 1.0, 2), (0.3, 1.0, 4), (0.25, 0.5, 2),
                                           (1.0, 1.0, 1), (0.2, 1.0, 5), (0.125, 2.0, 8)])
def test_zen_auto_steady_interval_closed_form(orc, lo, gamma, want):
    """Stationary magnitudes: the interval is ceil(gamma * important / unimportant)
    (SPEC S:449), capped by S_max (here 8 = N, so (0.125, 2) -> 16 is cut to 8)."""
    n, m = 16, 50
    M = _auto_model(orc, n, m, 100000, N=8, smax=8, gamma=gamma)
    G = _two_level(n, m, M.layers[0].k, 1.0, lo)
    P = np.zeros((n, m), np.float32)
    for t in range(24):
        M.step(t, [G], [P])
    iv = M.intervals()
    assert want == min(8, math.ceil(gamma / lo - 1e-9))
    # windows never cross a refresh (every 8 steps)
    full = [want] * (8 // want) + ([8 % want] if 8 % want else [])
    assert iv == full * 3, iv


def test_zen_auto_zero_stream_never_triggers(orc):
    """a zero gradient stream never triggers; windows end only at the cap and
    before refreshes."""
    n, m = 8, 40
    M = _auto_model(orc, n, m, 100000, N=6, smax=4, gamma=1.0)
    P = np.zeros((n, m), np.float32)
    G = np.zeros((n, m), np.float32)
    for t in range(12):
        M.step(t, [G], [P])
    assert M.intervals() == [4, 2, 4, 2]


def test_zen_auto_unimportant_zero_never_triggers(orc):
    """unimportant columns zero, important nonzero -> no trigger regardless of
    steps (only the refresh boundary ends the window)."""
    n, m = 8, 40
    M = _auto_model(orc, n, m, 100000, N=10, smax=10, gamma=1e-6)
    G = _two_level(n, m, M.layers[0].k, 3.0, 0.0)
    P = np.zeros((n, m), np.float32)
    for t in range(20):
        M.step(t, [G], [P])
    assert M.intervals() == [10, 10]


def test_zen_auto_monotone_in_unimportant_magnitude(orc):
    """with a fixed important part, larger unimportant norms never delay the
    trigger (random stream, important columns kept on top)."""
    rng = np.random.default_rng(70)
    n, m = 12, 60
    base = [rng.standard_normal((n, m)).astype(np.float32) for _ in range(16)]
    firsts = []
    for scale in (0.5, 1.0, 2.0, 4.0, 8.0):
        M = _auto_model(orc, n, m, 100000, N=16, smax=16, gamma=1.0)
        k = M.layers[0].k
        P = np.zeros((n, m), np.float32)
        for t in range(16):
            G = base[t] * np.float32(scale)
            G[:, :k] = base[t][:, :k] + np.float32(8.0)
            M.step(t, [G], [P])
        firsts.append(M.ends[0])
    assert firsts == sorted(firsts, reverse=True) and firsts[0] > firsts[-1], firsts


def test_zen_auto_huge_gamma_is_the_fixed_schedule(orc):
    """gamma -> infinity: windows end only at S_max (= S), so Zen-auto reduces to the fixed
    S-step schedule -- selection, moments, parameters (with f1), compact blocks and both
    accumulators bit-identical to stepping OracleLayer with fixed windows."""
    import synth
    n, m, N, S = 24, 96, 4, 2
    Ms = _auto_model(orc, n, m, 100000, N=N, smax=S, gamma=1e300, cpu_update=True, layers=2)
    Fs = [orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=N, accum_interval=S, cpu_update=True)
          for _ in range(2)]
    PA = [synth.param(n, m, layer=i, dtype="fp32") for i in range(2)]
    PB = [p.copy() for p in PA]
    for t in range(9):
        Gs = [synth.grad(n, m, i, t, synth.col_scale_at(m, t, i), dtype="fp32") for i in range(2)]
        outs = Ms.step(t, Gs, PA)
        for i in range(2):
            assert np.array_equal(outs[i], Fs[i].step(t, Gs[i], PB[i]))
            assert np.array_equal(PA[i], PB[i]) and np.array_equal(Ms.layers[i].acc[0], Fs[i].acc[0])
            assert np.array_equal(Ms.layers[i].acc[1], Fs[i].acc[1])
    assert Ms.intervals() == [2, 2, 2, 2]


def test_zen_auto_cpu_update_uses_the_window_length(orc):
    """f1 under Zen-auto: the CPU update happens exactly at the window end Zen-auto picks
    (ratio 0.25, gamma = 1 -> L = 4), once, and moves every unimportant column by the
    bias-corrected step-1 amount -lr*g/(|g|+eps).  At g = 0.25 >> eps that move is
    scale-invariant, so this pins WHEN the update lands and the step count, not the 1/L
    factor; ``test_f1_zen_auto_window_length_factor_in_the_eps_regime`` pins the factor."""
    n, m = 16, 64
    M = _auto_model(orc, n, m, 100000, N=8, smax=8, gamma=1.0, cpu_update=True)
    k = M.layers[0].k
    G = _two_level(n, m, k, 1.0, 0.25)
    P = np.zeros((n, m), np.float32)
    for t in range(3):
        M.step(t, [G], [P])
        assert np.all(P[:, k:] == 0.0)
    M.step(3, [G], [P])
    assert M.ends == [3]
    assert np.allclose(P[:, k:], -1e-3 * 0.25 / (0.25 + 1e-8), rtol=1e-6)
    assert M.layers[0].th[k:].tolist() == [1] * (m - k)


def test_zen_auto_pools_channels_over_the_model(orc):
    """R21: the important / unimportant means are over every column of the model (pooled),
    not averages of per-layer means.  Layer A: 16x40 with 4 important columns of 1.0 and 36
    unimportant of 0.5; layer B: 16x10 with 1 important column of 1.0 and 9 unimportant of
    0.0625.  Per-channel L2 norms: important 4, unimportant 2 (A) and 0.25 (B); pooled
    unimportant mean u = (36*2 + 9*0.25)/45 = 1.65, i = 4: with gamma = 1 the window ends
    when A = s*u >= 4, i.e. at s = 3 (s*u = 4.95; s = 2 gives 3.3).  (Averaging the two
    layers' means instead would give u = 1.125 -> s = 4.)"""
    n = 16
    LA = orc.OracleLayer(n=n, m=40, ratio_ppm=100000, refresh_interval=16, accum_interval=16)
    LB = orc.OracleLayer(n=n, m=10, ratio_ppm=100000, refresh_interval=16, accum_interval=16)
    assert LA.k == 4 and LB.k == 1
    M = orc.OracleModel([LA, LB], auto_gamma=1.0)
    GA = np.full((n, 40), 0.5, np.float32)
    GA[:, :4] = 1.0
    GB = np.full((n, 10), 0.0625, np.float32)
    GB[:, 0] = 1.0
    PA, PB = np.zeros((n, 40), np.float32), np.zeros((n, 10), np.float32)
    for t in range(9):
        M.step(t, [GA, GB], [PA, PB])
    assert M.intervals() == [3, 3, 3]
    A, i, u = M.stats[0]
    assert abs(u - (36 * 2 + 9 * 0.25) / 45) < 1e-12 and abs(i - 4.0) < 1e-12


# ------------------------------------------------------------------ f1: the 1/S factor of P:527
# AdamW is invariant to the scale of its gradient except through eps (and through an L2
# weight-decay term), so the factor 1/S of P:527 (theta^(c) -= alpha * (1/S) * sum over the
# window) is only visible where |g| is comparable to eps or where wd*p is added to g.  These
# pins sit in those regimes, with closed forms evaluated in double.
_TINY = 2.0 ** -27          # ~7.45e-9, comparable to eps = 1e-8; dyadic, so window sums are exact


def _step1_move(g, lr=1e-3, eps=1e-8):
    """Bias-corrected first AdamW step from zero moments: -lr * g / (|g| + eps)."""
    return -lr * g / (abs(g) + eps)


def test_f1_window_average_in_the_eps_regime(orc):
    """Fixed S = 2, constant unselected gradient g = 2^-27 ~ eps: the flush uses acc / S = g,
    so the move is -lr*g/(g+eps) = -4.27e-4; using the window SUM (2g) would move by
    -lr*2g/(2g+eps) = -5.98e-4 (reading R18)."""
    n, m = 4, 10
    G = np.full((n, m), _TINY, np.float32)
    G[:, 0] = 9.0                                      # column 0 selected (k = 1)
    P = np.zeros((n, m), np.float32)
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=2, accum_interval=2, cpu_update=True)
    L.step(0, G, P)
    L.step(1, G, P)
    want = _step1_move(_TINY)
    assert abs(want - _step1_move(2 * _TINY)) > 0.3 * abs(want)     # the regime separates the two
    assert np.allclose(P[:, 1:], want, rtol=1e-5, atol=0)


def test_f1_window_average_with_l2_weight_decay(orc):
    """Non-decoupled weight decay adds wd*p to the window average (O6 with g = acc/S):
    g' = 0.25 + 0.5 * (-0.75) = -0.125, so the first flush moves p UP by lr; with the window
    sum (0.5) g' = +0.125 and p would move down (P:527 + R8's L2 mode)."""
    n, m = 3, 8
    G = np.full((n, m), 0.25, np.float32)
    G[:, 0] = 9.0
    P = np.full((n, m), -0.75, np.float32)
    hp = orc.AdamHP(lr=1e-3, weight_decay=0.5, decoupled=0)
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=125000, refresh_interval=2, accum_interval=2, hp=hp, cpu_update=True)
    L.step(0, G, P)
    assert np.all(P[:, 1:] == np.float32(-0.75))
    L.step(1, G, P)
    want = -0.75 + _step1_move(0.25 + 0.5 * -0.75)     # = -0.75 + lr (to 1e-7 relative)
    assert np.allclose(P[:, 1:], want, rtol=1e-6, atol=0)
    assert np.all(P[:, 1:] > -0.75)


def test_f1_zen_auto_window_length_factor_in_the_eps_regime(orc):
    """Zen-auto with N = S_max = 8, gamma = 0.75 on a constant stream of tiny gradients
    (important 4*2^-27, unimportant 2^-27: per-channel ratio 0.25).  The decision ends a
    window after L = 3 steps (3 * 0.25 >= 0.75); windows are t = 0..2, 3..5, and 6..7, the
    last cut to L = 2 by the refresh at t = 8.  Each flush averages with its OWN length
    (P:527 with S = L, reading R21), so every flush sees g = 2^-27 and, with constant g, every
    AdamW step moves by -lr*g/(|g|+eps) (m_hat = g, v_hat = g^2).  Dividing by S_max would
    feed 3g/8, 3g/8, g/4; not dividing would feed 3g, 3g, 2g -- both change P."""
    n, m = 16, 64
    M = _auto_model(orc, n, m, 100000, N=8, smax=8, gamma=0.75, cpu_update=True)
    k = M.layers[0].k
    G = _two_level(n, m, k, 4 * _TINY, _TINY)
    P = np.zeros((n, m), np.float32)
    step = _step1_move(_TINY)
    for t in range(3):
        M.step(t, [G], [P])
    assert M.ends == [2]
    assert np.allclose(P[:, k:], step, rtol=1e-5, atol=0)
    for t in range(3, 8):
        M.step(t, [G], [P])
    assert M.intervals() == [3, 3, 2]
    assert np.allclose(P[:, k:], 3 * step, rtol=1e-5, atol=0)
    assert M.layers[0].th[k:].tolist() == [3] * (m - k)


# ------------------------------------------------------------------ f4 (ii): lagged selection (reading R24)
def _spike(n, m, col, big=8.0):
    G = np.full((n, m), 0.125, np.float32)
    G[:, col] = big
    return G


def test_lagged_refresh_ranks_by_the_previous_step(orc):
    """N = 2, k = 1: the step before the refresh at t = 2 has its large column at 5, the
    refresh step itself at 9.  A lagged selection (R24) picks 5; the plain one picks 9.  The
    first refresh (t = 0) has no earlier step and picks its own step's column (3)."""
    n, m = 4, 10
    seq = [_spike(n, m, 3), _spike(n, m, 5), _spike(n, m, 9), _spike(n, m, 9)]
    A = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=2, accum_interval=2, lagged=True)
    B = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=2, accum_interval=2)
    PA, PB = np.zeros((n, m), np.float32), np.zeros((n, m), np.float32)
    picks = []
    for t, G in enumerate(seq):
        A.step(t, G, PA)
        B.step(t, G, PB)
        picks.append((A.idx.tolist(), B.idx.tolist()))
    assert picks[0] == ([3], [3]) and picks[1] == ([3], [3])
    assert picks[2] == ([5], [9]) and picks[3] == ([5], [9])
    # column 5 enters at t = 2 and takes two AdamW steps on the constant g = 0.125 of steps 2
    # and 3 (closed form: each moves by -lr*g/(|g|+eps)); its step count is 2
    assert np.allclose(PA[:, 5], 2 * (-1e-3 * 0.125 / (0.125 + 1e-8)), rtol=1e-5) and A.steps.tolist() == [2]


def test_lagged_equals_plain_on_a_constant_stream(orc):
    """With G_t = G_{t-1} for all t the lagged ranking is the plain one: selection, moments,
    parameters, compact blocks and accumulators identical (N = 3, several refreshes)."""
    import synth
    n, m = 32, 96
    e = synth.col_scale_init(m, 0)
    G = synth.grad(n, m, 0, 0, e, dtype="fp32")
    A = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=3, accum_interval=3, lagged=True)
    B = orc.OracleLayer(n=n, m=m, ratio_ppm=100000, refresh_interval=3, accum_interval=3)
    PA = synth.param(n, m, 0, dtype="fp32")
    PB = PA.copy()
    for t in range(10):
        assert np.array_equal(A.step(t, G, PA), B.step(t, G, PB))
        assert np.array_equal(A.idx, B.idx) and np.array_equal(A.M, B.M) and np.array_equal(PA, PB)


def test_lagged_N1_uses_the_previous_step_every_step(orc):
    """N = 1: every step refreshes, each from the previous step's norms (k = 1)."""
    n, m = 4, 8
    cols = [1, 6, 2, 7, 0]
    L = orc.OracleLayer(n=n, m=m, ratio_ppm=125000, refresh_interval=1, accum_interval=1, lagged=True)
    P = np.zeros((n, m), np.float32)
    got = []
    for t, c in enumerate(cols):
        L.step(t, _spike(n, m, c), P)
        got.append(int(L.idx[0]))
    assert got == [1, 1, 6, 2, 7]
