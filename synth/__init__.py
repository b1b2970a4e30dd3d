"""Seeded synthetic inputs for the ZenFlow hot path (numpy twin of synth/synth.cu).

This module holds NO arithmetic of the method (no norms, selection, Adam,
compaction or accumulation).  It only draws the inputs both sides consume:
gradients G_t, initial parameters p_0, and the per-column scale state that
gives the gradients the column-concentrated, temporally-local structure the
paper reports (P:204 top-1% of grads ~ 88.9% of norm^2; P:296-303 columns
carry the large gradients; P:326-328 the important channels persist).  The
recipe is DESIGN.md §4 (SURVEY §8(d) "Synthetic value distribution"):

* counter-based SplitMix64: ``h = mix(stream_key(seed, tag, layer, step) + e)``
  with ``e`` the GLOBAL row-major element index ``i*m + j`` (so row shards of a
  matrix concatenate to the single-GPU matrix);
* ``z = sum of the four 16-bit chunks of h - 131070`` (Irwin-Hall(4), an
  integer in [-131070, 131070], std ~ 37837.2);
* column scale exponent ``e_j = clamp(round(2.885 * z / 37837.2), -24, 24)``
  (log-normal scale with sigma = 2 in natural-log units, as a power of two),
  redrawn each step with probability ~0.03% (``low32(h) < 1288490``).  Calibrated to the
  paper's temporal locality (fig. ratention_rate: the top-10% channels of a step keep
  "over 95% of the top-1% gradients across 100 iterations"): with i.i.d. values inside fixed
  column scales the fixed channel set keeps ~(1-p)^t of the top-1% elements after t steps, so
  p = 0.03% gives ~0.97 at t = 99 (tools/retention_sweep.py measures it).  SPEC S:151 proposes
  1% for its desk-scale simulator; that retains only ~0.35 after 100 steps;
* ``G[i][j] = round_to_dtype(z * 2^(e_j - 26))`` -- exact in fp32 (an 18-bit
  integer times a power of two), then ONE round-to-nearest-even to bf16;
* ``p0[i][j] = round_to_dtype(z * 2^-22)``;
* tie-heavy mode: ``G[i][j] = ((h mod 5) - 2) * 2^-8`` (many equal norms).

Both this file and synth.cu implement the same integer recipe, so the GPU
generator's output is bit-identical to this one (tests/test_synth.py).
"""
from __future__ import annotations

import numpy as np

SEED = 0x250512242
MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)
TAG_GRAD, TAG_SCALE, TAG_REDRAW, TAG_PARAM, TAG_TIE = 1, 2, 3, 4, 5
REDRAW_THRESHOLD = 1288490   # ~0.03% of 2^32 (calibrated to P:328, see the module doc)
E_MIN, E_MAX = -24, 24

_GOLD = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_K_TAG = 0xD1B54A32D192ED03
_K_LAYER = 0xABC98388FB8FAC03
_K_STEP = 0x8CB92BA72F3D8DD7


def _mix_py(x: int) -> int:
    x &= 0xFFFFFFFFFFFFFFFF
    z = (x + _GOLD) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * _M1) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * _M2) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def stream_key(seed: int, tag: int, layer: int, step: int) -> int:
    """64-bit key of one (tag, layer, step) stream."""
    x = (seed ^ ((tag * _K_TAG) & 0xFFFFFFFFFFFFFFFF) ^ ((layer * _K_LAYER) & 0xFFFFFFFFFFFFFFFF)
         ^ ((step * _K_STEP) & 0xFFFFFFFFFFFFFFFF))
    return _mix_py(x)


def _mix_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(_GOLD)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        return z ^ (z >> np.uint64(31))


def _hash(key: int, e: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return _mix_np(np.uint64(key) + e.astype(np.uint64))


def _ih4(h: np.ndarray) -> np.ndarray:
    m16 = np.uint64(0xFFFF)
    s = (h & m16) + ((h >> np.uint64(16)) & m16) + ((h >> np.uint64(32)) & m16) + ((h >> np.uint64(48)) & m16)
    return s.astype(np.int64) - 131070


def _scale_exp_from_z(z: np.ndarray) -> np.ndarray:
    # round-half-up(z * 2885 / 37837200) in exact integer arithmetic, then clamp
    num = z * 2885 + 18918600
    e = np.floor_divide(num, 37837200)
    return np.clip(e, E_MIN, E_MAX).astype(np.int8)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns (inputs are finite here)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))
    return (u >> np.uint64(16)).astype(np.uint16)


def _finish(vals_f32: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return f32_to_bf16_bits(vals_f32)
    if dtype == "fp32":
        return vals_f32.astype(np.float32)
    raise ValueError(dtype)


def col_scale_init(m: int, layer: int, seed: int = SEED) -> np.ndarray:
    """Column-scale exponents at step 0 (int8 [m])."""
    h = _hash(stream_key(seed, TAG_SCALE, layer, 0), np.arange(m, dtype=np.uint64))
    return _scale_exp_from_z(_ih4(h))


def col_scale_advance(e: np.ndarray, step: int, layer: int, seed: int = SEED) -> np.ndarray:
    """Exponents at ``step`` (>0) from those at ``step-1``: each column is redrawn w.p. ~0.03% (REDRAW_THRESHOLD / 2^32)."""
    m = e.shape[0]
    j = np.arange(m, dtype=np.uint64)
    hr = _hash(stream_key(seed, TAG_REDRAW, layer, step), j)
    redraw = (hr & np.uint64(0xFFFFFFFF)) < np.uint64(REDRAW_THRESHOLD)
    hn = _hash(stream_key(seed, TAG_SCALE, layer, step), j)
    return np.where(redraw, _scale_exp_from_z(_ih4(hn)), e).astype(np.int8)


def col_scale_at(m: int, step: int, layer: int, seed: int = SEED) -> np.ndarray:
    e = col_scale_init(m, layer, seed)
    for t in range(1, step + 1):
        e = col_scale_advance(e, t, layer, seed)
    return e


def grad(n: int, m: int, layer: int, step: int, scale_exp: np.ndarray, dtype: str = "bf16",
         row0: int = 0, m_total: int | None = None, seed: int = SEED) -> np.ndarray:
    """Rows [row0, row0+n) of the m-column gradient of ``layer`` at ``step``."""
    i = np.arange(row0, row0 + n, dtype=np.uint64)[:, None]
    j = np.arange(m, dtype=np.uint64)[None, :]
    h = _hash(stream_key(seed, TAG_GRAD, layer, step), i * np.uint64(m) + j)
    z = _ih4(h).astype(np.float32)
    scale = np.ldexp(np.float32(1.0), scale_exp.astype(np.int32) - 26).astype(np.float32)
    return _finish(z * scale[None, :], dtype)


def grad_tie(n: int, m: int, layer: int, step: int, dtype: str = "bf16", row0: int = 0,
             seed: int = SEED) -> np.ndarray:
    """Tie-heavy gradient: values in {-2..2} * 2^-8."""
    i = np.arange(row0, row0 + n, dtype=np.uint64)[:, None]
    j = np.arange(m, dtype=np.uint64)[None, :]
    h = _hash(stream_key(seed, TAG_TIE, layer, step), i * np.uint64(m) + j)
    v = (h % np.uint64(5)).astype(np.int64) - 2
    return _finish(v.astype(np.float32) * np.float32(2.0 ** -8), dtype)


def param(n: int, m: int, layer: int, dtype: str = "bf16", row0: int = 0, seed: int = SEED) -> np.ndarray:
    i = np.arange(row0, row0 + n, dtype=np.uint64)[:, None]
    j = np.arange(m, dtype=np.uint64)[None, :]
    h = _hash(stream_key(seed, TAG_PARAM, layer, 0), i * np.uint64(m) + j)
    return _finish(_ih4(h).astype(np.float32) * np.float32(2.0 ** -22), dtype)


# ------------------------------------------------------------ model shapes
def llama2_7b_linears():
    """Every nn.Linear weight of Llama-2-7B as (name, n=out, m=in) [R1, R16]."""
    out = []
    for L in range(32):
        for nm in ("q_proj", "k_proj", "v_proj", "o_proj"):
            out.append((f"layers.{L}.attn.{nm}", 4096, 4096))
        out.append((f"layers.{L}.mlp.gate_proj", 11008, 4096))
        out.append((f"layers.{L}.mlp.up_proj", 11008, 4096))
        out.append((f"layers.{L}.mlp.down_proj", 4096, 11008))
    out.append(("lm_head", 32000, 4096))
    return out


def llama2_13b_linears():
    out = []
    for L in range(40):
        for nm in ("q_proj", "k_proj", "v_proj", "o_proj"):
            out.append((f"layers.{L}.attn.{nm}", 5120, 5120))
        out.append((f"layers.{L}.mlp.gate_proj", 13824, 5120))
        out.append((f"layers.{L}.mlp.up_proj", 13824, 5120))
        out.append((f"layers.{L}.mlp.down_proj", 5120, 13824))
    out.append(("lm_head", 32000, 5120))
    return out


def gpt2_small_linears():
    """GPT-2 small linears in nn.Linear [out, in] orientation [R1]; lm_head tied to wte."""
    out = []
    for L in range(12):
        out.append((f"h.{L}.attn.c_attn", 2304, 768))
        out.append((f"h.{L}.attn.c_proj", 768, 768))
        out.append((f"h.{L}.mlp.c_fc", 3072, 768))
        out.append((f"h.{L}.mlp.c_proj", 768, 3072))
    out.append(("lm_head", 50257, 768))
    return out


MODELS = {"llama2-7b": llama2_7b_linears, "llama2-13b": llama2_13b_linears, "gpt2-small": gpt2_small_linears}
