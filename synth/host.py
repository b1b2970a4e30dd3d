"""ctypes binding of synth/libzfsynth_host.so: the host C twin of the numpy generator
(synth/__init__.py), bit-identical to it and ~20x faster -- used where full-size inputs
must be generated on the host (the CPU-oracle timing in bench.py)."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import SEED

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth_host.c")
_LIB = os.path.join(_HERE, "libzfsynth_host.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O3", "-fPIC", "-shared", "-ffp-contract=off", "-o", _LIB + ".tmp", _SRC,
                               "-lm"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i64, i32, u64, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p
        _lib.synth_host_col_scale_init.argtypes = [vp, i64, i32, u64]
        _lib.synth_host_col_scale_advance.argtypes = [vp, i64, i32, i64, u64]
        _lib.synth_host_grad.argtypes = [vp, ctypes.c_int, i64, i64, i64, i64, i32, i64, vp, u64]
        _lib.synth_host_param.argtypes = [vp, ctypes.c_int, i64, i64, i64, i64, i32, u64]
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def col_scale_at(m: int, step: int, layer: int, seed: int = SEED) -> np.ndarray:
    e = np.empty(m, np.int8)
    lib().synth_host_col_scale_init(_p(e), m, layer, seed)
    for t in range(1, step + 1):
        lib().synth_host_col_scale_advance(_p(e), m, layer, t, seed)
    return e


def grad(n: int, m: int, layer: int, step: int, scale_exp: np.ndarray, dtype: str = "bf16", row0: int = 0,
         seed: int = SEED) -> np.ndarray:
    out = np.empty((n, m), np.uint16 if dtype == "bf16" else np.float32)
    e = np.ascontiguousarray(scale_exp, np.int8)
    lib().synth_host_grad(_p(out), 1 if dtype == "bf16" else 0, n, m, m, row0, layer, step, _p(e), seed)
    return out


def param(n: int, m: int, layer: int, dtype: str = "bf16", row0: int = 0, seed: int = SEED) -> np.ndarray:
    out = np.empty((n, m), np.uint16 if dtype == "bf16" else np.float32)
    lib().synth_host_param(_p(out), 1 if dtype == "bf16" else 0, n, m, m, row0, layer, seed)
    return out
