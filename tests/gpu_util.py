"""Helpers shared by the GPU parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np
import torch


def to_np(t: torch.Tensor) -> np.ndarray:
    """Host copy; bf16 as uint16 bit patterns (the oracle's bf16 representation)."""
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16).copy()
    return t.numpy().copy()


def from_np(a: np.ndarray, device="cuda") -> torch.Tensor:
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).to(device)
    return torch.from_numpy(a.copy()).to(device)


def assert_bits_equal(got: np.ndarray, want: np.ndarray, what: str):
    assert got.shape == want.shape, (what, got.shape, want.shape)
    g, w = got.view(np.uint8), want.view(np.uint8)
    if not np.array_equal(g, w):
        bad = np.nonzero(got.reshape(-1).view(got.dtype) != want.reshape(-1))[0]
        raise AssertionError(f"{what}: {bad.size} elements differ, first at {bad[:5]}: "
                             f"{got.reshape(-1)[bad[:5]]} vs {want.reshape(-1)[bad[:5]]}")


def bf16_ulp_diff(a: np.ndarray, b: np.ndarray) -> int:
    """Max distance in bf16 ulps between two bf16 bit-pattern arrays (same sign assumed near)."""
    def key(x):
        x = x.astype(np.int32)
        return np.where(x & 0x8000, -(x & 0x7FFF), x & 0x7FFF)
    return int(np.max(np.abs(key(a) - key(b)))) if a.size else 0


def assert_close_rel(got: np.ndarray, want: np.ndarray, rtol: float, what: str):
    got = got.astype(np.float64)
    want = want.astype(np.float64)
    err = np.abs(got - want)
    lim = rtol * np.abs(want)
    if not np.all(err <= lim):
        i = np.argmax(err - lim)
        raise AssertionError(f"{what}: rel err {err.flat[i] / max(abs(want.flat[i]), 1e-300):.3g} at {i} "
                             f"(got {got.flat[i]!r}, want {want.flat[i]!r}) > {rtol}")


def selection_ok(gpu_idx: np.ndarray, orc_idx: np.ndarray, orc_norms: np.ndarray, tol: float = 1e-5):
    """Reading R3: index sets bit-exact, except boundary swaps between columns whose
    (oracle) norms are within tol of each other and of the k-th value."""
    a, b = set(gpu_idx.tolist()), set(orc_idx.tolist())
    assert len(gpu_idx) == len(orc_idx) and list(gpu_idx) == sorted(gpu_idx) and len(a) == len(gpu_idx)
    if a == b:
        return 0
    only_g, only_o = sorted(a - b), sorted(b - a)
    kth = np.min(orc_norms[list(b)])
    for j in only_g + only_o:
        assert abs(float(orc_norms[j]) - float(kth)) <= tol * max(float(kth), 1e-30), \
            f"non-boundary selection difference at column {j}: {orc_norms[j]} vs k-th {kth}"
    return len(only_g)
