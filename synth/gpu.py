"""ctypes binding of synth/libzfsynth.so (GPU twin of the numpy generator in synth/__init__.py)."""
from __future__ import annotations

import ctypes
import os

import torch

from . import SEED

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libzfsynth.so")
if not os.path.exists(_LIB):
    raise ImportError(f"{_LIB} not built; run `python -m paper_2505_12242_b200._build`")
lib = ctypes.CDLL(_LIB)
_i64, _i32, _u64, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p
lib.synth_col_scale_init.argtypes = [_vp, _i64, _i32, _u64, _vp]
lib.synth_col_scale_advance.argtypes = [_vp, _i64, _i32, _i64, _u64, _vp]
lib.synth_grad.argtypes = [_vp, ctypes.c_int, _i64, _i64, _i64, _i64, _i32, _i64, _vp, _u64, _vp]
lib.synth_grad_tie.argtypes = [_vp, ctypes.c_int, _i64, _i64, _i64, _i64, _i32, _i64, _u64, _vp]
lib.synth_param.argtypes = [_vp, ctypes.c_int, _i64, _i64, _i64, _i64, _i32, _u64, _vp]
for f in (lib.synth_col_scale_init, lib.synth_col_scale_advance, lib.synth_grad, lib.synth_grad_tie, lib.synth_param):
    f.restype = ctypes.c_int


def _s():
    return torch.cuda.current_stream().cuda_stream


def _dt(t):
    return 1 if t.dtype == torch.bfloat16 else 0


def _ok(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed: cuda error {rc}")


class ColScale:
    """Device-resident per-column scale exponents of one layer (advanced step by step)."""

    def __init__(self, m: int, layer: int, seed: int = SEED):
        self.m, self.layer, self.seed, self.step = m, layer, seed, 0
        self.e = torch.empty(m, dtype=torch.int8, device="cuda")
        _ok(lib.synth_col_scale_init(self.e.data_ptr(), m, layer, seed, _s()), "col_scale_init")

    def advance_to(self, step: int):
        assert step >= self.step
        while self.step < step:
            self.step += 1
            _ok(lib.synth_col_scale_advance(self.e.data_ptr(), self.m, self.layer, self.step, self.seed, _s()),
                "col_scale_advance")


def fill_grad(out: torch.Tensor, layer: int, step: int, scale: ColScale, row0: int = 0, seed: int = SEED):
    n, m = out.shape
    if n == 0:
        return
    _ok(lib.synth_grad(out.data_ptr(), _dt(out), n, m, out.stride(0), row0, layer, step, scale.e.data_ptr(), seed,
                       _s()), "synth_grad")


def fill_grad_tie(out: torch.Tensor, layer: int, step: int, row0: int = 0, seed: int = SEED):
    n, m = out.shape
    if n == 0:
        return
    _ok(lib.synth_grad_tie(out.data_ptr(), _dt(out), n, m, out.stride(0), row0, layer, step, seed, _s()),
        "synth_grad_tie")


def fill_param(out: torch.Tensor, layer: int, row0: int = 0, seed: int = SEED):
    n, m = out.shape
    if n == 0:
        return
    _ok(lib.synth_param(out.data_ptr(), _dt(out), n, m, out.stride(0), row0, layer, seed, _s()), "synth_param")
