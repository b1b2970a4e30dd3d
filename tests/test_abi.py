"""The C-ABI library: loads, exports every symbol include/zf.h declares, and
rejects bad arguments synchronously (ZF_EINVAL) -- all without a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def zf():
    from paper_2505_12242_b200 import _build
    _build.build()
    from paper_2505_12242_b200 import zf as z
    return z


def _declared():
    src = open(os.path.join(ROOT, "include", "zf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(zf_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(zf):
    names = _declared()
    assert len(names) >= 18
    for n in names:
        assert hasattr(zf.lib, n), n
    assert set(names) == set(zf.SYMBOLS)


def test_version_and_k_for_closed_form(zf):
    assert zf.version() == 100
    assert zf.k_for(4096, 100000) == 410 and zf.k_for(4096, 10000) == 41
    assert zf.k_for(13824, 10000) == 139 and zf.k_for(100, 70000) == 7
    assert zf.lib.zf_k_for(0, 1000) == -1 and zf.lib.zf_k_for(10, 0) == -1 and zf.lib.zf_k_for(10, 1000001) == -1


def test_status_strings(zf):
    for s in range(7):
        assert zf.lib.zf_status_string(s)
    assert b"unknown" in zf.lib.zf_status_string(99)


FAKE = 0x10000  # never dereferenced: validation fails before anything is enqueued


def test_column_norms_validation(zf):
    L = zf.lib
    assert L.zf_column_norms(FAKE, 1, 0, 8, 8, FAKE, None, None) == zf.ZF_EINVAL
    assert L.zf_column_norms(FAKE, 1, 4, 8, 7, FAKE, None, None) == zf.ZF_EINVAL      # ld < m
    assert L.zf_column_norms(FAKE, 7, 4, 8, 8, FAKE, None, None) == zf.ZF_EINVAL      # dtype
    assert L.zf_column_norms(None, 1, 4, 8, 8, FAKE, None, None) == zf.ZF_EINVAL
    assert L.zf_column_norms(FAKE, 1, 4, 8, 8, None, None, None) == zf.ZF_EINVAL
    assert b"ld" in L.zf_last_error() or b"NULL" in L.zf_last_error()


def test_topk_validation(zf):
    L = zf.lib
    assert L.zf_topk_columns(FAKE, 0, 1, FAKE, None) == zf.ZF_EINVAL                  # empty
    assert L.zf_topk_columns(FAKE, 10, 0, FAKE, None) == zf.ZF_EINVAL
    assert L.zf_topk_columns(FAKE, 10, 11, FAKE, None) == zf.ZF_EINVAL
    assert b"k" in L.zf_last_error()


def test_adam_and_compact_validation(zf):
    L = zf.lib
    hp = zf.adam_params()
    bad = zf.adam_params(beta1=1.0)
    assert L.zf_selective_adam(FAKE, 1, 8, FAKE, 1, 8, 4, 8, FAKE, 0, FAKE, FAKE, FAKE, ctypes.byref(hp),
                               None) == zf.ZF_EINVAL
    assert L.zf_selective_adam(FAKE, 1, 8, FAKE, 1, 8, 4, 8, FAKE, 2, FAKE, FAKE, FAKE, ctypes.byref(bad),
                               None) == zf.ZF_EINVAL
    assert L.zf_compact_unselected(FAKE, 1, 4, 8, 8, FAKE, 9, FAKE, None) == zf.ZF_EINVAL
    assert L.zf_compact_unselected(FAKE, 1, 4, 8, 8, FAKE, 2, FAKE + 2, None) == zf.ZF_EINVAL  # misaligned out


def test_create_validation(zf):
    L = zf.lib
    descs = (zf.LayerDesc * 1)()
    descs[0].n, descs[0].m, descs[0].ld_grad, descs[0].ld_param = 4, 8, 8, 8
    cfg = zf.Config()
    cfg.grad_dtype = cfg.param_dtype = zf.ZF_BF16
    cfg.topk_ppm, cfg.refresh_interval, cfg.accum_interval = 100000, 4, 4
    cfg.adam = zf.adam_params()
    h = ctypes.c_void_p()
    cfg.topk_ppm = 0
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 1, 0, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL
    cfg.topk_ppm = 100000
    cfg.host_accumulate, cfg.offload = 1, 0
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 1, 0, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL
    cfg.offload, cfg.refresh_interval, cfg.accum_interval = 1, 6, 4                  # N % S != 0
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 1, 0, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL
    cfg.refresh_interval = 4
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 2, 2, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL  # rank >= world
    cfg.auto_gamma = -1.0                                                              # Zen-auto gamma < 0
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 1, 0, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL
    cfg.auto_gamma, cfg.host_accumulate = 1.0, 0                                       # Zen-auto needs H1
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 1, 0, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL
    assert b"auto_gamma" in L.zf_last_error()
    cfg.auto_gamma = 0.0
    cfg.host_accumulate = 1
    cfg.host_stages = 17                                                               # > 16 staging slots
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 1, 0, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL
    assert b"host_stages" in L.zf_last_error()
    cfg.host_stages = 0
    cfg.refresh_group_mb = -1
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 1, 0, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL
    cfg.refresh_group_mb = 64                                                          # grouped refresh: world 1 only
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 2, 0, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL
    assert b"refresh_group_mb" in L.zf_last_error()
    cfg.refresh_group_mb = 0
    cfg.lagged_selection, cfg.auto_gamma = 1, 1.0                                      # lag + Zen-auto exclusive
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 1, 0, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL
    cfg.lagged_selection, cfg.auto_gamma = 0, 0.0
    descs[0].ld_grad = 7
    assert L.zf_create(descs, 1, ctypes.byref(cfg), 1, 0, None, 0, ctypes.byref(h)) == zf.ZF_EINVAL
    assert not h.value


def test_null_context_calls(zf):
    """Context calls reject a NULL context with ZF_EINVAL (no GPU needed)."""
    L = zf.lib
    a, b = ctypes.c_int64(), ctypes.c_int64()
    assert L.zf_host_stats(None, ctypes.byref(a), ctypes.byref(b)) == zf.ZF_EINVAL
    buf = ctypes.create_string_buffer(64 * 2)
    assert L.zf_peer_handle(None, buf) == zf.ZF_EINVAL
    assert L.zf_peer_open(None, buf) == zf.ZF_EINVAL
    assert L.zf_sync(None) == zf.ZF_EINVAL


def test_product_does_not_import_oracle():
    """The product package and the oracle share no code and never import each other."""
    pkg = os.path.join(ROOT, "paper_2505_12242_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(//|#).*", "", txt).replace("oracle/", ""), f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".cpp")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert "import paper_2505_12242_b200" not in txt and "zf_internal" not in txt and "zf.h" not in txt


def test_struct_layouts_match_the_header(zf, tmp_path):
    """The ctypes mirrors of zf_config / zf_adam_params / zf_layer_desc have the header's field
    order, offsets and sizes (a silent mismatch would misconfigure every context): a small C
    program including include/zf.h prints offsetof / sizeof for each field."""
    import shutil
    import subprocess
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {"zf_config": zf.Config, "zf_adam_params": zf.AdamParams, "zf_layer_desc": zf.LayerDesc}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "zf.h"', "int main(void) {"]
    for cname, cls in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _t in cls._fields_:
            lines.append(f'  printf("{cname}.{fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                          check=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[f"{cname} size"]) == ctypes.sizeof(cls), cname
        for fname, _t in cls._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(cls, fname).offset, (cname, fname)
