"""Python side of the CPU ORACLE (ctypes over oracle/liboracle.so + step orchestration).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product package ``paper_2505_12242_b200`` never imports it, and it
never imports the product package.

Arrays: fp32 data are ``np.float32``; bf16 data are ``np.uint16`` holding the
bf16 bit patterns.  All arithmetic happens in ``zf_oracle.cpp``; this file only
marshals arguments and sequences the steps of the method in the paper's order:

* refresh (every N steps, "cache and reuse selected channel indices"):
  column norms (O1) -> top-k (O3) -> moment remap (O5, reading R7);
* selective AdamW on the selected columns (O6);
* compaction of the unselected columns (O7);
* accumulation into the active buffer of a double-buffered pair, zeroed at the
  start of each S-step window and sealed at its end (O8).

``OracleLayer.step`` has the semantics ``zf_step`` implements.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "zf_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

F32, BF16 = 0, 1

_i64, _i32, _f32, _f64, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_float, ctypes.c_double, ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile the oracle (g++ -O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.oracle_bf16_round.argtypes = [_f32]; L.oracle_bf16_round.restype = _f32
        L.oracle_k_for.argtypes = [_i64, _i32]; L.oracle_k_for.restype = _i64
        L.oracle_column_norms.argtypes = [_vp, ctypes.c_int, _i64, _i64, _i64, _vp]
        L.oracle_column_norms.restype = ctypes.c_int
        L.oracle_column_norms_f64.argtypes = [_vp, ctypes.c_int, _i64, _i64, _i64, _vp]
        L.oracle_column_norms_f64.restype = None
        L.oracle_topk.argtypes = [_vp, _i64, _i64, _vp]; L.oracle_topk.restype = ctypes.c_int
        L.oracle_column_map.argtypes = [_vp, _i64, _i64, _vp, _vp]; L.oracle_column_map.restype = None
        L.oracle_remap.argtypes = [_i64, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp]
        L.oracle_remap.restype = None
        L.oracle_selective_adamw.argtypes = [_vp, ctypes.c_int, _i64, _vp, ctypes.c_int, _i64, _i64,
                                             _vp, _i64, _vp, _vp, _vp, _f64, _f64, _f64, _f64, _f64,
                                             ctypes.c_int]
        L.oracle_selective_adamw.restype = None
        L.oracle_compact.argtypes = [_vp, ctypes.c_int, _i64, _i64, _i64, _vp, _i64, _vp]
        L.oracle_compact.restype = None
        L.oracle_accumulate.argtypes = [_vp, _vp, ctypes.c_int, _i64]; L.oracle_accumulate.restype = None
        L.oracle_to_bf16.argtypes = [_vp, _vp, _i64]; L.oracle_to_bf16.restype = None
        L.oracle_channel_norm_sums.argtypes = [_vp, _i64, _vp, _i64, _vp]
        L.oracle_channel_norm_sums.restype = None
        L.oracle_zen_auto_decide.argtypes = [ctypes.POINTER(_f64), ctypes.POINTER(_i64), ctypes.c_int, _f64, _i64,
                                             _f64, _i64, _f64, _i64, ctypes.c_int]
        L.oracle_zen_auto_decide.restype = ctypes.c_int
    return _lib


def _dt(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return F32
    if a.dtype == np.uint16:
        return BF16
    raise TypeError(f"oracle arrays are float32 or uint16(bf16 bits), got {a.dtype}")


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- primitives
def bf16_round(x: float) -> float:
    return float(lib().oracle_bf16_round(float(x)))


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns (left shift by 16)."""
    return (h.astype(np.uint32) << 16).view(np.float32)


def as_f32(a: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f32(a) if a.dtype == np.uint16 else a.astype(np.float32)


def to_bf16(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty(x.shape, np.uint16)
    lib().oracle_to_bf16(_p(x), _p(out), x.size)
    return out


def k_for(m: int, ratio_ppm: int) -> int:
    return int(lib().oracle_k_for(m, ratio_ppm))


def column_norms(G: np.ndarray) -> np.ndarray:
    G = np.ascontiguousarray(G)
    n, m = G.shape
    out = np.empty(m, np.float32)
    bad = lib().oracle_column_norms(_p(G), _dt(G), n, m, m, _p(out))
    if bad:
        raise FloatingPointError("non-finite gradient (SPEC S:44 rejects)")
    return out


def column_norms_f64(G: np.ndarray) -> np.ndarray:
    G = np.ascontiguousarray(G)
    n, m = G.shape
    out = np.empty(m, np.float64)
    lib().oracle_column_norms_f64(_p(G), _dt(G), n, m, m, _p(out))
    return out


def topk(norms: np.ndarray, k: int) -> np.ndarray:
    norms = np.ascontiguousarray(norms, dtype=np.float32)
    m = norms.shape[0]
    if m == 0:
        raise ValueError("empty norms vector (S:108)")
    if not 1 <= k <= m:
        raise ValueError("k out of range")
    idx = np.empty(k, np.int32)
    if lib().oracle_topk(_p(norms), m, k, _p(idx)):
        raise FloatingPointError("non-finite norm")
    return idx


def column_map(idx: np.ndarray, m: int):
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    slot = np.empty(m, np.int32)
    upos = np.empty(m, np.int32)
    lib().oracle_column_map(_p(idx), idx.shape[0], m, _p(slot), _p(upos))
    return slot, upos


def remap(n, idx_old, m_old, v_old, step_old, idx_new):
    k = idx_new.shape[0]
    m_new = np.empty((n, k), np.float32)
    v_new = np.empty((n, k), np.float32)
    step_new = np.empty(k, np.int32)
    lib().oracle_remap(n, _p(idx_old), idx_old.shape[0], _p(m_old), _p(v_old), _p(step_old),
                       _p(idx_new), k, _p(m_new), _p(v_new), _p(step_new))
    return m_new, v_new, step_new


@dataclass
class AdamHP:
    """Reading R8: PyTorch AdamW defaults; the paper gives lr 1e-5, wd 0.
    Real-valued (double) hyper-parameters; derived fp32 constants are rounded once."""
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0
    decoupled: int = 1


def selective_adamw(P: np.ndarray, G: np.ndarray, idx: np.ndarray, M: np.ndarray, V: np.ndarray,
                    step: np.ndarray, hp: AdamHP) -> None:
    """In place on P (selected columns), M, V, step."""
    n, m = G.shape
    assert P.shape == G.shape and M.shape == V.shape == (n, idx.shape[0]) and step.shape == idx.shape
    lib().oracle_selective_adamw(_p(P), _dt(P), P.shape[1], _p(G), _dt(G), m, n, _p(idx), idx.shape[0],
                                 _p(M), _p(V), _p(step), hp.lr, hp.beta1, hp.beta2, hp.eps,
                                 hp.weight_decay, int(hp.decoupled))


def compact(G: np.ndarray, idx: np.ndarray) -> np.ndarray:
    G = np.ascontiguousarray(G)
    n, m = G.shape
    k = idx.shape[0]
    out = np.empty((n, m - k), G.dtype)
    lib().oracle_compact(_p(G), _dt(G), n, m, m, _p(np.ascontiguousarray(idx, np.int32)), k, _p(out))
    return out


def accumulate(acc: np.ndarray, stage: np.ndarray) -> None:
    assert acc.dtype == np.float32 and acc.size == stage.size
    lib().oracle_accumulate(_p(acc), _p(np.ascontiguousarray(stage)), _dt(stage), acc.size)


def shard_rows(n: int, world: int, rank: int):
    """Row-wise contiguous partition, near-equal, remainder to the earliest shards
    (4096x4096 into 4 -> 1024-row shards; 5 rows into 2 -> 3+2)."""
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


# -------------------------------------------------------------- step driver
@dataclass
class OracleLayer:
    """One weight matrix under the method (the state zf_step keeps for it).

    refresh_interval = N (selection refreshed iff t % N == 0, [R6]);
    accum_interval = S (window length of the CPU-side accumulation).
    """
    n: int
    m: int
    ratio_ppm: int
    refresh_interval: int = 4
    accum_interval: int = 4
    hp: AdamHP = field(default_factory=AdamHP)
    cpu_update: bool = False   # f1: deferred CPU AdamW on the unselected columns (reading R18)
    warmup: int = 0            # f2: tau synchronous warm-up steps with k = m (reading R20)
    lagged: bool = False       # f4 (ii): a refresh after the first selects by the previous step's norms (R24)
    lag_norms: np.ndarray | None = None
    idx: np.ndarray | None = None
    M: np.ndarray | None = None
    V: np.ndarray | None = None
    steps: np.ndarray | None = None
    acc: list | None = None
    last_norms: np.ndarray | None = None
    last_out: np.ndarray | None = None
    master: np.ndarray | None = None     # f1: fp32 master of theta^(c) [n, m] (valid on unselected columns)
    Mh: np.ndarray | None = None         # f1: host moments [n, m]
    Vh: np.ndarray | None = None
    th: np.ndarray | None = None         # f1: host step count per column [m]

    @property
    def k(self) -> int:
        return k_for(self.m, self.ratio_ppm)

    def step(self, t: int, G: np.ndarray, P: np.ndarray, idx_override: np.ndarray | None = None,
             window: tuple | None = None):
        """One step of the hot path for this matrix at global step t.

        idx_override: use this selection instead of the oracle's own top-k on a
        refresh step (parity protocol O10: downstream steps are compared on the
        GPU's selection, so a tolerated boundary swap never cascades).

        window: None for the fixed schedule (windows [wS, (w+1)S) of the regular
        step index, O8); or (w, first) from ``OracleModel`` under Zen-auto (reading
        R21): accumulate into buffer w % 2, zeroing it first if ``first``; the window's
        end (and the f1 update) is then decided by the caller (``end_window``)."""
        if t < self.warmup:
            return self._warmup_step(G, P)
        t -= self.warmup                    # R20: the regular schedule starts at step tau
        k = self.k
        if self.cpu_update:
            assert self.refresh_interval % self.accum_interval == 0, "R18: refresh only at window starts"
        if t % self.refresh_interval == 0 or self.idx is None:
            # R24 (f4 ii, "cache and reuse selected channel indices"): with a lagged
            # selection every refresh but the first ranks the columns by the norms of the step
            # before it; the first (no earlier regular step) by its own gradient's
            self.last_norms = self.lag_norms if (self.lagged and self.lag_norms is not None) else column_norms(G)
            new_idx = topk(self.last_norms, k) if idx_override is None else np.asarray(idx_override, np.int32)
            old_idx = self.idx
            if self.idx is None:
                self.M = np.zeros((self.n, k), np.float32)
                self.V = np.zeros((self.n, k), np.float32)
                self.steps = np.zeros(k, np.int32)
            else:
                self.M, self.V, self.steps = remap(self.n, self.idx, self.M, self.V, self.steps, new_idx)
            self.idx = new_idx
            if self.cpu_update:
                self._migrate(old_idx, new_idx, P)
        selective_adamw(P, G, self.idx, self.M, self.V, self.steps, self.hp)
        out = compact(G, self.idx)
        if self.lagged and (t + 1) % self.refresh_interval == 0:
            self.lag_norms = column_norms(G)            # the next refresh's ranking (R24)
        S = self.accum_interval
        if self.acc is None:
            self.acc = [np.zeros((self.n, self.m - k), np.float32) for _ in range(2)]
        w, first = (t // S, t % S == 0) if window is None else window
        a = w % 2
        if first:
            self.acc[a][...] = 0.0
        accumulate(self.acc[a], out)
        self.last_out = out
        if window is None and (t + 1) % S == 0:
            self.end_window(w, S, P)
        return out

    def end_window(self, w: int, length: int, P: np.ndarray):
        """Seal window w (buffer w % 2) after `length` steps; with f1 its average gradient
        updates theta^(c) (reading R18; 1/S of P:527 with S = the window's length)."""
        if self.cpu_update:
            self._deferred_update(self.acc[w % 2], P, length)

    # ---------------------------------------------------------------- f2 warm-up
    def _warmup_step(self, G, P):
        """f2 / reading R20 ("synchronous updates (i.e., no staleness) during the
        initial tau warm-up steps"): every column is important (k = m): the step is plain
        AdamW (O6) on the whole matrix, nothing is offloaded.  The state is kept as a
        selection of all m columns, so the first regular refresh (step tau) remaps it by R7:
        columns selected at tau keep their moments and step counts."""
        n, m = self.n, self.m
        if self.idx is None:
            self.idx = np.arange(m, dtype=np.int32)
            self.M = np.zeros((n, m), np.float32)
            self.V = np.zeros((n, m), np.float32)
            self.steps = np.zeros(m, np.int32)
        selective_adamw(P, G, self.idx, self.M, self.V, self.steps, self.hp)
        out = np.empty((n, 0), G.dtype)
        self.last_out = out
        return out

    # ---------------------------------------------------------------- f1
    def _unselected(self):
        mask = np.ones(self.m, bool)
        mask[self.idx] = False
        return np.nonzero(mask)[0].astype(np.int32)

    def _migrate(self, old_idx, new_idx, P):
        """Reading R18 at a refresh: a column entering the CPU-updated set (unselected now,
        selected before or first step) takes the current parameter value as its fp32
        master, with zero host moments and step count (as R7 does on the GPU side);
        a column leaving it keeps nothing."""
        if self.master is None:
            self.master = np.zeros((self.n, self.m), np.float32)
            self.Mh = np.zeros((self.n, self.m), np.float32)
            self.Vh = np.zeros((self.n, self.m), np.float32)
            self.th = np.zeros(self.m, np.int32)
        was_cpu = np.zeros(self.m, bool)
        if old_idx is not None:
            was_cpu[:] = True
            was_cpu[old_idx] = False
        now_cpu = np.ones(self.m, bool)
        now_cpu[new_idx] = False
        entering = np.nonzero(now_cpu & ~was_cpu)[0]
        self.master[:, entering] = as_f32(P[:, entering])
        self.Mh[:, entering] = 0.0
        self.Vh[:, entering] = 0.0
        self.th[entering] = 0

    def _deferred_update(self, acc, P, length=None):
        """f1 / reading R18: at the end of an S-step window, theta^(c) (the window's
        unselected columns) takes one AdamW step (formula O6) with the window's
        average gradient acc / S (theta^(c) -= alpha * (1/S) * sum of the
        window's gradients, here through AdamW), on the fp32 master with host
        moments; the parameter then holds the master rounded to its dtype."""
        unsel = self._unselected()
        S = self.accum_interval if length is None else length
        g_avg = acc / np.float32(S)                            # one IEEE fp32 division
        Gfull = np.zeros((self.n, self.m), np.float32)
        Gfull[:, unsel] = g_avg
        Mc = np.ascontiguousarray(self.Mh[:, unsel])
        Vc = np.ascontiguousarray(self.Vh[:, unsel])
        tc = np.ascontiguousarray(self.th[unsel])
        selective_adamw(self.master, Gfull, unsel, Mc, Vc, tc, self.hp)
        self.Mh[:, unsel] = Mc
        self.Vh[:, unsel] = Vc
        self.th[unsel] = tc
        if P.dtype == np.uint16:
            P[:, unsel] = to_bf16(self.master[:, unsel])
        else:
            P[:, unsel] = self.master[:, unsel]

    def sealed(self, t: int):
        """The accumulator sealed by the window that ended at or before step t."""
        t -= self.warmup
        S = self.accum_interval
        w = t // S if (t + 1) % S == 0 else t // S - 1
        return None if w < 0 else self.acc[w % 2]


# ------------------------------------------------------------ f2: Zen-auto (R21)
def channel_norm_sums(norms: np.ndarray, idx: np.ndarray):
    """O11: (sum of sqrt(norm) over the selected columns, over the unselected columns)."""
    norms = np.ascontiguousarray(norms, np.float32)
    idx = np.ascontiguousarray(idx, np.int32)
    out = np.zeros(2, np.float64)
    lib().oracle_channel_norm_sums(_p(norms), norms.shape[0], _p(idx), idx.shape[0], _p(out))
    return float(out[0]), float(out[1])


class ZenAuto:
    """O12 state: Zen-auto's adaptive update interval (reading R21)."""

    def __init__(self, gamma: float, smax: int):
        assert gamma > 0 and smax >= 1
        self.gamma, self.smax = float(gamma), int(smax)
        self.A = ctypes.c_double(0.0)
        self.len = ctypes.c_int64(0)
        self.first = True

    def decide(self, sel_sum, sel_cnt, unsel_sum, unsel_cnt, force_end: bool) -> bool:
        end = bool(lib().oracle_zen_auto_decide(ctypes.byref(self.A), ctypes.byref(self.len), int(self.first),
                                                sel_sum, sel_cnt, unsel_sum, unsel_cnt, self.gamma, self.smax,
                                                int(force_end)))
        self.first = end
        return end


class OracleModel:
    """All weight matrices of a model under the method, stepped together (``zf_step``
    over a context's layers).  Without ``auto_gamma`` each layer follows its own fixed
    S-step windows (identical to stepping the ``OracleLayer`` objects one by one).
    With ``auto_gamma`` > 0 (Zen-auto, f2, reading R21) the accumulation windows of
    every layer end together, when the model-wide Zen-auto decision (O11/O12, on every
    step's column norms) says so, after accum_interval (= S_max) steps, or before a
    refresh; with f1 each window's CPU update uses its own length as S."""

    def __init__(self, layers: list, auto_gamma: float = 0.0):
        self.layers = layers
        l0 = layers[0]
        for l in layers:
            assert (l.refresh_interval, l.accum_interval, l.warmup) == \
                (l0.refresh_interval, l0.accum_interval, l0.warmup)
        self.N, self.S, self.tau = l0.refresh_interval, l0.accum_interval, l0.warmup
        self.auto = ZenAuto(auto_gamma, self.S) if auto_gamma > 0 else None
        self.w = 0                 # index of the current window
        self.w_len = 0
        self.ends: list = []       # global step t of every window end (Zen-auto: the interval history)
        self.stats: list = []      # per regular step: (A, i, u) of the decision

    def step(self, t: int, Gs: list, Ps: list, idx_overrides: list | None = None):
        outs = []
        if t < self.tau or self.auto is None:
            for li, l in enumerate(self.layers):
                outs.append(l.step(t, Gs[li], Ps[li], None if idx_overrides is None else idx_overrides[li]))
            if t >= self.tau and (t - self.tau + 1) % self.S == 0:
                self.ends.append(t)
            return outs
        tr = t - self.tau
        first = self.auto.first
        sel = [0.0, 0, 0.0, 0]
        for li, l in enumerate(self.layers):
            outs.append(l.step(t, Gs[li], Ps[li], None if idx_overrides is None else idx_overrides[li],
                               window=(self.w, first)))
            a, b = channel_norm_sums(column_norms(Gs[li]), l.idx)
            sel[0] += a
            sel[1] += l.k
            sel[2] += b
            sel[3] += l.m - l.k
        force = (tr + 1) % self.N == 0
        end = self.auto.decide(sel[0], sel[1], sel[2], sel[3], force)
        u = sel[2] / sel[3] if sel[3] else 0.0
        i = sel[0] / sel[1] if sel[1] else 0.0
        self.stats.append((self.auto.A.value, i, u))
        if end:
            length = int(self.auto.len.value)
            for li, l in enumerate(self.layers):
                l.end_window(self.w, length, Ps[li])
            self.ends.append(t)
            self.w += 1
        return outs

    def intervals(self):
        """Window lengths so far (the Zen-auto interval history)."""
        out, prev = [], self.tau - 1
        for e in self.ends:
            out.append(e - prev)
            prev = e
        return out
