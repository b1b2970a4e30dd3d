"""Thin ctypes binding of libzf.so (include/zf.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libzf.so; this module
only converts torch tensors to pointers/sizes and checks status codes.  There
is no fallback: if libzf.so is missing or cannot be loaded, importing this
module raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libzf.so")

ZF_OK, ZF_EINVAL, ZF_ENONFINITE, ZF_ECUDA, ZF_ENCCL, ZF_ENOMEM, ZF_ESTATE = range(7)
ZF_FP32, ZF_BF16 = 0, 1

SYMBOLS = ["zf_status_string", "zf_last_error", "zf_version", "zf_k_for", "zf_column_norms", "zf_topk_columns",
           "zf_selective_adam", "zf_compact_unselected", "zf_nccl_unique_id", "zf_create", "zf_step", "zf_sync",
           "zf_selected", "zf_norms", "zf_optimizer_state", "zf_compact_buffer", "zf_host_accumulator", "zf_device_accumulator", "zf_window_log", "zf_set_host_allreduce", "zf_set_lr",
           "zf_kernel_launches", "zf_profile", "zf_profile_read", "zf_params_changed", "zf_host_stats", "zf_peer_handle", "zf_peer_open", "zf_destroy"]


class ZFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class AdamParams(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("weight_decay", ctypes.c_double), ("decoupled", ctypes.c_int32)]


class LayerDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64), ("ld_grad", ctypes.c_int64),
                ("ld_param", ctypes.c_int64)]


class Config(ctypes.Structure):
    _fields_ = [("grad_dtype", ctypes.c_int32), ("param_dtype", ctypes.c_int32), ("topk_ppm", ctypes.c_int32),
                ("refresh_interval", ctypes.c_int32), ("accum_interval", ctypes.c_int32), ("adam", AdamParams),
                ("offload", ctypes.c_int32), ("host_accumulate", ctypes.c_int32), ("host_threads", ctypes.c_int32),
                ("cpu_update", ctypes.c_int32), ("warmup_steps", ctypes.c_int32),
                ("auto_gamma", ctypes.c_float), ("state_offload", ctypes.c_int32),
                ("device_accumulate", ctypes.c_int32), ("cpu_update_async", ctypes.c_int32),
                ("param_subset", ctypes.c_int32), ("lagged_selection", ctypes.c_int32),
                ("host_stages", ctypes.c_int32), ("refresh_group_mb", ctypes.c_int32)]


if not os.path.exists(_LIB_PATH):
    raise ImportError(f"libzf.so not built at {_LIB_PATH}; run `python -m paper_2505_12242_b200._build` "
                      "(there is no CPU fallback)")
lib = ctypes.CDLL(_LIB_PATH)

_i64, _i32, _vp, _st = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int
_pp = ctypes.POINTER(ctypes.c_void_p)
lib.zf_status_string.argtypes = [_i32]; lib.zf_status_string.restype = ctypes.c_char_p
lib.zf_last_error.argtypes = []; lib.zf_last_error.restype = ctypes.c_char_p
lib.zf_version.argtypes = []; lib.zf_version.restype = _i32
lib.zf_k_for.argtypes = [_i64, _i32]; lib.zf_k_for.restype = _i64
lib.zf_column_norms.argtypes = [_vp, _st, _i64, _i64, _i64, _vp, _vp, _vp]; lib.zf_column_norms.restype = _st
lib.zf_topk_columns.argtypes = [_vp, _i64, _i64, _vp, _vp]; lib.zf_topk_columns.restype = _st
lib.zf_selective_adam.argtypes = [_vp, _st, _i64, _vp, _st, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _vp,
                                  ctypes.POINTER(AdamParams), _vp]
lib.zf_selective_adam.restype = _st
lib.zf_compact_unselected.argtypes = [_vp, _st, _i64, _i64, _i64, _vp, _i64, _vp, _vp]
lib.zf_compact_unselected.restype = _st
lib.zf_nccl_unique_id.argtypes = [_vp]; lib.zf_nccl_unique_id.restype = _st
lib.zf_create.argtypes = [ctypes.POINTER(LayerDesc), _i32, ctypes.POINTER(Config), _i32, _i32, _vp, _i32,
                          ctypes.POINTER(_vp)]
lib.zf_create.restype = _st
lib.zf_step.argtypes = [_vp, _i64, _pp, _pp, _vp]; lib.zf_step.restype = _st
lib.zf_sync.argtypes = [_vp]; lib.zf_sync.restype = _st
lib.zf_selected.argtypes = [_vp, _i32, ctypes.POINTER(_vp), ctypes.POINTER(_i64)]; lib.zf_selected.restype = _st
lib.zf_norms.argtypes = [_vp, _i32, ctypes.POINTER(_vp)]; lib.zf_norms.restype = _st
lib.zf_optimizer_state.argtypes = [_vp, _i32, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
lib.zf_optimizer_state.restype = _st
lib.zf_compact_buffer.argtypes = [_vp, _i32, ctypes.POINTER(_vp), ctypes.POINTER(_i64), ctypes.POINTER(_vp)]
lib.zf_compact_buffer.restype = _st
lib.zf_host_accumulator.argtypes = [_vp, _i32, _i32, ctypes.POINTER(_vp), ctypes.POINTER(_i64),
                                    ctypes.POINTER(_i64)]
lib.zf_host_accumulator.restype = _st
_pd = ctypes.POINTER(ctypes.c_double)
lib.zf_window_log.argtypes = [_vp, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i32), _pd, _pd, _pd,
                              ctypes.POINTER(_i64)]
lib.zf_window_log.restype = _st
lib.zf_device_accumulator.argtypes = [_vp, _i32, _i32, ctypes.POINTER(_vp), ctypes.POINTER(_i64)]
lib.zf_device_accumulator.restype = _st
HOST_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.POINTER(ctypes.c_float), ctypes.c_int64, ctypes.c_void_p)
lib.zf_set_host_allreduce.argtypes = [_vp, HOST_ALLREDUCE_FN, _vp]
lib.zf_set_host_allreduce.restype = _st
lib.zf_set_lr.argtypes = [_vp, ctypes.c_double]; lib.zf_set_lr.restype = _st
lib.zf_params_changed.argtypes = [_vp]; lib.zf_params_changed.restype = _st
lib.zf_kernel_launches.argtypes = [_vp]; lib.zf_kernel_launches.restype = _i64
lib.zf_peer_handle.argtypes = [_vp, _vp]; lib.zf_peer_handle.restype = _st
lib.zf_peer_open.argtypes = [_vp, _vp]; lib.zf_peer_open.restype = _st
lib.zf_host_stats.argtypes = [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]; lib.zf_host_stats.restype = _st
lib.zf_destroy.argtypes = [_vp]; lib.zf_destroy.restype = _st
lib.zf_profile.argtypes = [_vp, _i32]; lib.zf_profile.restype = _st
lib.zf_profile_read.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64)]
lib.zf_profile_read.restype = _st


def _check(st: int, what: str):
    if st != ZF_OK:
        raise ZFError(st, f"{what}: {lib.zf_status_string(st).decode()}: {lib.zf_last_error().decode()}")


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return ZF_BF16
    if t.dtype == torch.float32:
        return ZF_FP32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _mat(t: torch.Tensor):
    assert t.dim() == 2 and t.stride(1) == 1, "row-major 2-D tensor with unit column stride required"
    return t.data_ptr(), t.shape[0], t.shape[1], t.stride(0)


def k_for(m: int, ratio_ppm: int) -> int:
    return int(lib.zf_k_for(m, ratio_ppm))


def version() -> int:
    return int(lib.zf_version())


# ------------------------------------------------------------ stateless primitives
def zf_column_norms(G: torch.Tensor, norms: torch.Tensor, nonfinite: torch.Tensor | None = None, stream=None):
    p, n, m, ld = _mat(G)
    assert norms.dtype == torch.float32 and norms.numel() >= m
    _check(lib.zf_column_norms(p, _dt(G), n, m, ld, norms.data_ptr(),
                               nonfinite.data_ptr() if nonfinite is not None else None, _stream(stream)),
           "zf_column_norms")
    return norms


def zf_topk_columns(norms: torch.Tensor, k: int, idx: torch.Tensor, stream=None):
    assert norms.dtype == torch.float32 and idx.dtype == torch.int32
    _check(lib.zf_topk_columns(norms.data_ptr(), norms.numel(), k, idx.data_ptr(), _stream(stream)),
           "zf_topk_columns")
    return idx


def adam_params(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, decoupled=True) -> AdamParams:
    return AdamParams(lr, beta1, beta2, eps, weight_decay, int(bool(decoupled)))


def zf_selective_adam(P: torch.Tensor, G: torch.Tensor, idx: torch.Tensor, exp_avg: torch.Tensor,
                      exp_avg_sq: torch.Tensor, step: torch.Tensor, hp: AdamParams, stream=None):
    pp, n, m, ldp = _mat(P)
    gp, n2, m2, ldg = _mat(G)
    assert (n, m) == (n2, m2)
    k = idx.numel()
    assert exp_avg.dtype == exp_avg_sq.dtype == torch.float32 and step.dtype == torch.int32
    assert exp_avg.numel() == n * k and exp_avg_sq.numel() == n * k and step.numel() == k
    _check(lib.zf_selective_adam(pp, _dt(P), ldp, gp, _dt(G), ldg, n, m, idx.data_ptr(), k, exp_avg.data_ptr(),
                                 exp_avg_sq.data_ptr(), step.data_ptr(), ctypes.byref(hp), _stream(stream)),
           "zf_selective_adam")


def zf_compact_unselected(G: torch.Tensor, idx: torch.Tensor, out: torch.Tensor, stream=None):
    gp, n, m, ld = _mat(G)
    k = idx.numel()
    assert out.dtype == G.dtype and out.numel() >= n * (m - k)
    _check(lib.zf_compact_unselected(gp, _dt(G), n, m, ld, idx.data_ptr(), k, out.data_ptr(), _stream(stream)),
           "zf_compact_unselected")
    return out


def zf_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.zf_nccl_unique_id(buf), "zf_nccl_unique_id")
    return buf.raw


# ------------------------------------------------------------ device views (zero-copy)
class _DevView:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _view(ptr: int, shape, torch_dtype) -> torch.Tensor:
    typestr = {torch.float32: "<f4", torch.int32: "<i4", torch.bfloat16: "<u2"}[torch_dtype]
    if any(int(d) == 0 for d in shape):
        # an empty view (a layer with no rows on this rank): its pointer may sit one past the
        # end of the library's block, which torch refuses to wrap; nothing to alias anyway
        return torch.empty(tuple(int(d) for d in shape), dtype=torch_dtype, device="cuda")
    t = torch.as_tensor(_DevView(ptr, shape, typestr), device="cuda")
    return t.view(torch.bfloat16) if torch_dtype == torch.bfloat16 else t


@dataclass
class LayerShape:
    n: int
    m: int
    ld_grad: int | None = None
    ld_param: int | None = None


class Context:
    """The stateful driver (zf_create / zf_step / zf_sync / zf_destroy)."""

    def __init__(self, layers, grad_dtype=torch.bfloat16, param_dtype=torch.bfloat16, topk_ratio_ppm=100000,
                 refresh_interval=4, accum_interval=4, adam: AdamParams | None = None, offload=False,
                 host_accumulate=False, host_threads=0, world=1, rank=0, nccl_id: bytes | None = None,
                 device: int | None = None, cpu_update=False, warmup_steps=0, auto_gamma=0.0,
                 state_offload=False, device_accumulate=False, host_allreduce=None, cpu_update_async=False,
                 param_subset=True, lagged_selection=False, host_stages=0, refresh_group_mb=0):
        self.layers = [l if isinstance(l, LayerShape) else LayerShape(*l) for l in layers]
        descs = (LayerDesc * len(self.layers))()
        for d, l in zip(descs, self.layers):
            d.n, d.m = l.n, l.m
            d.ld_grad = l.ld_grad or l.m
            d.ld_param = l.ld_param or l.m
        self.grad_dtype, self.param_dtype = grad_dtype, param_dtype
        cfg = Config()
        cfg.grad_dtype = ZF_BF16 if grad_dtype == torch.bfloat16 else ZF_FP32
        cfg.param_dtype = ZF_BF16 if param_dtype == torch.bfloat16 else ZF_FP32
        cfg.topk_ppm = topk_ratio_ppm
        cfg.refresh_interval = refresh_interval
        cfg.accum_interval = accum_interval
        cfg.adam = adam if adam is not None else adam_params()
        cfg.offload = int(offload)
        cfg.host_accumulate = int(host_accumulate)
        cfg.host_threads = host_threads
        cfg.cpu_update = int(cpu_update)
        cfg.warmup_steps = int(warmup_steps)
        cfg.auto_gamma = float(auto_gamma)
        cfg.state_offload = int(state_offload)
        cfg.device_accumulate = int(device_accumulate)
        cfg.cpu_update_async = int(cpu_update_async)
        cfg.param_subset = int(param_subset)
        cfg.lagged_selection = int(lagged_selection)
        cfg.host_stages = int(host_stages)
        cfg.refresh_group_mb = int(refresh_group_mb)
        self.cfg = cfg
        self.device = torch.cuda.current_device() if device is None else device
        h = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(lib.zf_create(descs, len(descs), ctypes.byref(cfg), world, rank, idbuf, self.device,
                             ctypes.byref(h)), "zf_create")
        self._h = h
        self.k = [k_for(l.m, topk_ratio_ppm) for l in self.layers]
        self._ar = None
        if host_allreduce is not None:
            # host_allreduce(np.ndarray float32 [count]) sums in place over the ranks (e.g. gloo)
            import numpy as np

            def _cb(buf, count, user):
                try:
                    host_allreduce(np.ctypeslib.as_array(buf, shape=(count,)))
                    return 0
                except Exception:  # noqa: BLE001 -- reported as ZF_ENCCL by zf_step
                    return 1
            self._ar = HOST_ALLREDUCE_FN(_cb)
            _check(lib.zf_set_host_allreduce(h, self._ar, None), "zf_set_host_allreduce")
        n = len(self.layers)
        self._gp = (ctypes.c_void_p * n)()
        self._pp = (ctypes.c_void_p * n)()

    def step(self, t: int, grads, params, stream=None):
        for i, (g, p) in enumerate(zip(grads, params)):
            self._gp[i] = g.data_ptr()
            self._pp[i] = p.data_ptr()
        _check(lib.zf_step(self._h, t, self._gp, self._pp, _stream(stream)), "zf_step")

    def step_ptrs(self, t: int, gptrs, pptrs, stream=None):
        """zf_step with raw device pointers (ctypes arrays) -- no per-call marshalling."""
        _check(lib.zf_step(self._h, t, gptrs, pptrs, _stream(stream)), "zf_step")

    def sync(self):
        _check(lib.zf_sync(self._h), "zf_sync")

    def params_changed(self):
        """param_subset: the caller wrote the parameters outside step(); the next step re-reads
        the selected columns from them."""
        _check(lib.zf_params_changed(self._h), "zf_params_changed")

    def set_lr(self, lr: float):
        _check(lib.zf_set_lr(self._h, lr), "zf_set_lr")

    def profile(self, enable: bool = True):
        _check(lib.zf_profile(self._h, int(enable)), "zf_profile")

    PHASES = ("k1_norms", "allreduce", "k2_topk", "k3_update", "d2h_step", "d2h_window", "k7_accumulate", "k3b_adam")

    def profile_read(self):
        """{phase: (summed ms, count)} since the last read (waits for the recorded events)."""
        ms = (ctypes.c_double * len(self.PHASES))()
        n = (ctypes.c_int64 * len(self.PHASES))()
        _check(lib.zf_profile_read(self._h, ms, n), "zf_profile_read")
        return {p: (ms[i], n[i]) for i, p in enumerate(self.PHASES)}

    def kernel_launches(self) -> int:
        return int(lib.zf_kernel_launches(self._h))

    def peer_handle(self) -> bytes:
        """This rank's 64-byte IPC handle of its norm-exchange region (f4 iii)."""
        buf = ctypes.create_string_buffer(64)
        _check(lib.zf_peer_handle(self._h, buf), "zf_peer_handle")
        return buf.raw

    def peer_open(self, handles) -> None:
        """Map the other ranks' exchange regions (handles: one 64-byte handle per rank, rank
        order); the norm exchange then runs over peer memory."""
        raw = b"".join(bytes(h) for h in handles)
        _check(lib.zf_peer_open(self._h, ctypes.create_string_buffer(raw, len(raw))), "zf_peer_open")

    def host_stats(self):
        """(H1 accumulation passes, steps they covered) so far."""
        a, b = _i64(), _i64()
        _check(lib.zf_host_stats(self._h, ctypes.byref(a), ctypes.byref(b)), "zf_host_stats")
        return int(a.value), int(b.value)

    # views of library-owned state (device tensors share memory with the library)
    def selected(self, layer: int) -> torch.Tensor:
        p, k = ctypes.c_void_p(), ctypes.c_int64()
        _check(lib.zf_selected(self._h, layer, ctypes.byref(p), ctypes.byref(k)), "zf_selected")
        return _view(p.value, (k.value,), torch.int32)

    def norms(self, layer: int) -> torch.Tensor:
        p = ctypes.c_void_p()
        _check(lib.zf_norms(self._h, layer, ctypes.byref(p)), "zf_norms")
        return _view(p.value, (self.layers[layer].m,), torch.float32)

    def optimizer_state(self, layer: int):
        a, b, s = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _check(lib.zf_optimizer_state(self._h, layer, ctypes.byref(a), ctypes.byref(b), ctypes.byref(s)),
               "zf_optimizer_state")
        n, k = self.layers[layer].n, self.selected(layer).numel()   # k = m during warm-up
        return (_view(a.value, (n, k), torch.float32), _view(b.value, (n, k), torch.float32),
                _view(s.value, (k,), torch.int32))

    def compact_buffer(self, layer: int) -> torch.Tensor:
        """Device compact block [n, m-k] (a strided view: rows are padded to 16 bytes)."""
        d, ld, h = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_void_p()
        _check(lib.zf_compact_buffer(self._h, layer, ctypes.byref(d), ctypes.byref(ld), ctypes.byref(h)),
               "zf_compact_buffer")
        n, mk = self.layers[layer].n, self.layers[layer].m - self.k[layer]
        return _view(d.value, (n, ld.value), self.grad_dtype)[:, :mk]

    def compact_host(self, layer: int):
        """numpy view of the pinned host copy (valid after sync()); bf16 as uint16 bits."""
        import numpy as np
        d, ld, h = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_void_p()
        _check(lib.zf_compact_buffer(self._h, layer, ctypes.byref(d), ctypes.byref(ld), ctypes.byref(h)),
               "zf_compact_buffer")
        if not h.value:
            return None
        n, mk = self.layers[layer].n, self.layers[layer].m - self.k[layer]
        ct = ctypes.c_uint16 if self.grad_dtype == torch.bfloat16 else ctypes.c_float
        arr = (ct * (n * ld.value)).from_address(h.value)
        return np.ctypeslib.as_array(arr).reshape(n, ld.value)[:, :mk]

    def host_accumulator(self, layer: int, which: int = 0):
        import numpy as np
        p, r, c = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib.zf_host_accumulator(self._h, layer, which, ctypes.byref(p), ctypes.byref(r), ctypes.byref(c)),
               "zf_host_accumulator")
        if not p.value:
            return None
        arr = (ctypes.c_float * (r.value * c.value)).from_address(p.value)
        return np.ctypeslib.as_array(arr).reshape(r.value, c.value)

    def device_accumulator(self, layer: int, which: int = 0):
        """device_accumulate: the fp32 device accumulator [n, m-k] (strided view), or None."""
        p, ld = ctypes.c_void_p(), ctypes.c_int64()
        _check(lib.zf_device_accumulator(self._h, layer, which, ctypes.byref(p), ctypes.byref(ld)),
               "zf_device_accumulator")
        if not p.value:
            return None
        n, mk = self.layers[layer].n, self.layers[layer].m - self.k[layer]
        return _view(p.value, (n, ld.value), torch.float32)[:, :mk]

    def window_log(self):
        """Accumulation-window log after sync(): list of (t, ended, A, imp, unimp) per regular
        step (Zen-auto decision inputs; NaN with fixed windows)."""
        n = ctypes.c_int64()
        _check(lib.zf_window_log(self._h, 0, None, None, None, None, None, ctypes.byref(n)), "zf_window_log")
        cnt = n.value
        t = (ctypes.c_int64 * max(cnt, 1))()
        e = (ctypes.c_int32 * max(cnt, 1))()
        A, i, u = ((ctypes.c_double * max(cnt, 1))() for _ in range(3))
        _check(lib.zf_window_log(self._h, cnt, t, e, A, i, u, ctypes.byref(n)), "zf_window_log")
        return [(t[q], bool(e[q]), A[q], i[q], u[q]) for q in range(cnt)]

    def close(self):
        if getattr(self, "_h", None):
            lib.zf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
