"""The C-ABI library loads on a CPU-only box and exports every symbol that
include/entmax_attn.h declares; host-side validation paths work without a GPU."""
import ctypes
import os
import re

import pytest

from paper_2502_12082_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in sorted(os.listdir(os.path.join(ROOT, "include")))
           if h.endswith(".h")]


def _declared():
    names = set()
    for h in HEADERS:
        src = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        names |= set(re.findall(r"\b(entmax_\w+)\s*\(", src))
    return sorted(names)


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("entmax_attn_fwd", "entmax_attn_bwd", "entmax_attn_block_size",
                 "entmax_attn_fwd_workspace_bytes", "entmax_attn_bwd_workspace_bytes",
                 "entmax_attn_status_string", "entmax_attn_last_error",
                 "entmax_rowwise_fwd", "entmax_rowwise_bwd"):
        assert must in names


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in _declared():
        assert hasattr(L, name), name


def test_status_strings_and_block_size():
    L = _lib.lib()
    assert L.entmax_attn_status_string(0) == b"ok"
    assert L.entmax_attn_status_string(3) == b"workspace too small"
    br, bc = ctypes.c_int32(), ctypes.c_int32()
    for d in (16, 32, 64, 128):
        for dt in (0, 1):
            br.value = bc.value = 0
            assert L.entmax_attn_block_size(d, dt, ctypes.byref(br), ctypes.byref(bc)) == 0
            assert (br.value, bc.value) == (128, 128)
    br.value = bc.value = -1
    assert L.entmax_attn_block_size(96, 0, ctypes.byref(br), ctypes.byref(bc)) == 2   # unsupported head dim
    assert L.entmax_attn_block_size(64, 7, ctypes.byref(br), ctypes.byref(bc)) == 1   # unknown dtype
    assert (br.value, bc.value) == (-1, -1)   # outputs untouched on error
    assert L.entmax_attn_block_size(64, 0, None, None) == 0


def test_workspace_sizes_scale_with_blocks():
    L = _lib.lib()
    s = _lib.Shape(4, 12, 8192, 64, 12 * 8192 * 64, 8192 * 64, 64)
    fw = L.entmax_attn_fwd_workspace_bytes(ctypes.byref(s), 0, 0)
    bw = L.entmax_attn_bwd_workspace_bytes(ctypes.byref(s), 0, 0)
    BH, T = 48, 64
    assert fw >= BH * T * 4 + BH * T * T * 4
    assert bw >= BH * 8192 * 4 + BH * T * 4 + BH * T * T * 4


@pytest.mark.parametrize("alpha,n_iter,status", [(1.0, 3, 1), (0.5, 3, 1), (2.5, 3, 2), (1.5, 0, 1)])
def test_fwd_rejects_bad_arguments_before_launch(alpha, n_iter, status):
    L = _lib.lib()
    s = _lib.Shape(1, 1, 256, 64, 256 * 64, 256 * 64, 64)
    fake = ctypes.c_void_p(0x10000)  # never dereferenced: validation fails first
    rc = L.entmax_attn_fwd(fake, fake, fake, ctypes.byref(s), 0, alpha, 0, n_iter, 0.0,
                           fake, fake, fake, fake, fake, fake, fake, 1 << 30, None)
    assert rc == status
    assert L.entmax_attn_last_error()


def test_fwd_rejects_small_workspace_and_bad_strides():
    L = _lib.lib()
    fake = ctypes.c_void_p(0x10000)
    s = _lib.Shape(1, 1, 256, 64, 256 * 64, 256 * 64, 64)
    rc = L.entmax_attn_fwd(fake, fake, fake, ctypes.byref(s), 0, 1.5, 0, 3, 0.0,
                           fake, fake, fake, fake, fake, fake, fake, 16, None)
    assert rc == _lib.ENTMAX_ERR_WORKSPACE
    bad = _lib.Shape(1, 1, 256, 64, 256 * 64, 256 * 64, 60)   # rows overlap
    rc = L.entmax_attn_fwd(fake, fake, fake, ctypes.byref(bad), 0, 1.5, 0, 3, 0.0,
                           fake, fake, fake, fake, fake, fake, fake, 1 << 30, None)
    assert rc == _lib.ENTMAX_ERR_INVALID_ARG
    s3 = _lib.Shape(1, 1, 256, 48, 256 * 48, 256 * 48, 48)    # d=48 has no kernel
    assert L.entmax_attn_impl_for(ctypes.byref(s3), 0) == -1


def test_binding_refuses_cpu_tensors():
    import torch
    import paper_2502_12082_b200 as P
    x = torch.zeros(1, 1, 128, 64, dtype=torch.bfloat16)
    with pytest.raises(RuntimeError):
        P.entmax_attn_fwd(x, x, x)


@pytest.mark.parametrize("alpha,n_iter,rows,n,ld,status", [
    (1.0, 3, 4, 64, 64, 1), (2.5, 3, 4, 64, 64, 2), (1.5, 0, 4, 64, 64, 1),
    (1.5, 3, 0, 64, 64, 1), (1.5, 3, 4, 0, 64, 1), (1.5, 3, 4, 64, 32, 1), (1.5, 3, 4, 63, 63, 1)])
def test_rowwise_rejects_bad_arguments_before_launch(alpha, n_iter, rows, n, ld, status):
    L = _lib.lib()
    fake = ctypes.c_void_p(0x10000)   # never dereferenced: validation fails first
    rc = L.entmax_rowwise_fwd(fake, rows, n, ld, 1, alpha, n_iter, 1, fake, None, None)
    assert rc == status
    assert L.entmax_attn_last_error().decode()


def test_rowwise_bwd_rejects_misaligned_pointer():
    L = _lib.lib()
    rc = L.entmax_rowwise_bwd(ctypes.c_void_p(0x10004), ctypes.c_void_p(0x10000), 2, 64, 64, 1, 1.5,
                              ctypes.c_void_p(0x10000), None)
    assert rc == 1


def test_unmasked_mode_partial_null_tables_rejected_before_launch():
    """mask / row_cnt / row_idx must be all set or all NULL (unmasked mode, NEXT-2)."""
    L = _lib.lib()
    s = _lib.Shape(1, 1, 256, 64, 256 * 64, 256 * 64, 64)
    fake = ctypes.c_void_p(0x10000)
    rc = L.entmax_attn_fwd(fake, fake, fake, ctypes.byref(s), 0, 1.5, 0, 3, 0.0,
                           fake, fake, fake, fake, None, fake, fake, 1 << 30, None)
    assert rc == 1 and b"all NULL" in L.entmax_attn_last_error()
    rc = L.entmax_attn_bwd(fake, fake, fake, fake, fake, fake, None, fake, None, ctypes.byref(s), 0, 1.5, 0, 0.0,
                           fake, fake, fake, fake, 1 << 30, None)
    assert rc == 1 and b"all NULL" in L.entmax_attn_last_error()


def test_pack_mask_validation():
    L = _lib.lib()
    assert L.entmax_attn_pack_mask(None, 4, 8, ctypes.c_void_p(0x10000), None) == 1
    assert L.entmax_attn_pack_mask(ctypes.c_void_p(0x10000), 0, 8, ctypes.c_void_p(0x10000), None) == 1


def test_too_many_heads_rejected_before_launch():
    L = _lib.lib()
    s = _lib.Shape(70000, 1, 128, 64, 128 * 64, 128 * 64, 64)
    fake = ctypes.c_void_p(0x10000)
    rc = L.entmax_attn_fwd(fake, fake, fake, ctypes.byref(s), 0, 1.5, 0, 3, 0.0,
                           fake, fake, fake, fake, fake, fake, fake, 1 << 40, None)
    assert rc == 2 and b"65535" in L.entmax_attn_last_error()


def test_no_cpu_fallback():
    """The product path never computes on the host: CPU tensors are rejected loudly."""
    import torch
    import paper_2502_12082_b200 as P
    x = torch.zeros(1, 1, 128, 64, dtype=torch.bfloat16)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.entmax_attn_fwd(x, x, x, 1.5, False, 3)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.entmax_rowwise_fwd(torch.zeros(4, 64), 1.5, 3)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.entmax_attention(x, x, x)
