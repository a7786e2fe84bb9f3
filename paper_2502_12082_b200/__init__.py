"""B200-native AdaSplash α-entmax attention (arXiv 2502.12082) — Python binding.

Thin marshalling layer over the C ABI in include/entmax_attn.h: every step of the hot
path runs in the CUDA kernels of libentmax_attn.so.  PyTorch supplies device memory, the
current CUDA stream and autograd plumbing only.  There is no CPU/eager fallback: when the
library or a CUDA device is missing the calls raise.

Public API (same names as the C ABI):
  entmax_attn_fwd(q, k, v, alpha, causal, n_iter, scale=None, training=True, masked=True) -> FwdResult
  entmax_attn_bwd(q, k, v, d_o, fwd: FwdResult, alpha, causal, scale=None) -> (dq, dk, dv)
  entmax_attention(q, k, v, alpha=1.5, causal=False, n_iter=3, scale=None, masked=True)  (autograd op)
    masked=False: the paper's unmasked variant (every visible block, no mask / lookup tables).
  entmax_rowwise_fwd(s, alpha, n_iter, halley=True) -> (p, tau)    (include/entmax_rowwise.h)
  entmax_rowwise_bwd(p, dp, alpha) -> ds
  entmax(s, alpha=1.5, n_iter=3, halley=True)  (autograd op over the last dimension)
q, k, v: [B, H, N, d] CUDA tensors, bf16 (tcgen05 path) or fp32 (SIMT fp32 path), same
strides, last dim contiguous.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import EntmaxAttnError, ENTMAX_BF16, ENTMAX_FP32

__all__ = ["entmax_attn_fwd", "entmax_attn_bwd", "entmax_attention", "block_size", "FwdResult",
           "EntmaxAttnError", "impl_for", "profile_enable", "profile_reset", "profile_collect",
           "workspace_bytes", "entmax_rowwise_fwd", "entmax_rowwise_bwd", "entmax", "pack_mask"]

_DT = {torch.bfloat16: ENTMAX_BF16, torch.float32: ENTMAX_FP32}


def block_size(d: int = 64, dtype=torch.bfloat16):
    """(B_r, B_c): mask / lookup-table granularity of the library for head dim d and dtype."""
    br, bc = ctypes.c_int32(), ctypes.c_int32()
    st = _lib.lib().entmax_attn_block_size(int(d), _DT[dtype], ctypes.byref(br), ctypes.byref(bc))
    _lib.check(st, "entmax_attn_block_size")
    return br.value, bc.value


def _shape(q: torch.Tensor) -> _lib.Shape:
    if q.dim() != 4:
        raise ValueError("expected [B, H, N, d] tensors")
    B, H, N, d = q.shape
    sb, sh, sn, sd = q.stride()
    if sd != 1:
        raise ValueError("last dimension must be contiguous")
    return _lib.Shape(B, H, N, d, sb, sh, sn)


def _check_inputs(*ts):
    q = ts[0]
    if not q.is_cuda:
        raise RuntimeError("entmax_attn: tensors must be CUDA tensors (no CPU fallback)")
    if q.dtype not in _DT:
        raise TypeError(f"unsupported dtype {q.dtype}")
    for t in ts[1:]:
        if t.shape != q.shape or t.stride() != q.stride() or t.dtype != q.dtype or t.device != q.device:
            raise ValueError("q, k, v (and o2, dO) must share shape, strides, dtype and device")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def impl_for(q: torch.Tensor) -> int:
    """1 = tcgen05 kernels, 0 = SIMT fp32 kernels, -1 = unsupported."""
    return _lib.lib().entmax_attn_impl_for(ctypes.byref(_shape(q)), _DT[q.dtype])


def workspace_bytes(q: torch.Tensor, causal: bool):
    L = _lib.lib()
    s = _shape(q)
    return (L.entmax_attn_fwd_workspace_bytes(ctypes.byref(s), _DT[q.dtype], int(causal)),
            L.entmax_attn_bwd_workspace_bytes(ctypes.byref(s), _DT[q.dtype], int(causal)))


@dataclass
class FwdResult:
    o: torch.Tensor        # [B,H,N,d]
    o2: torch.Tensor       # [B,H,N,d] fp32 contiguous, or None (inference)
    tau: torch.Tensor      # [B,H,N] fp32
    mask: torch.Tensor     # [B,H,T_r,T_c] uint8
    row_cnt: torch.Tensor  # [B,H,T_r] int32
    row_idx: torch.Tensor  # [B,H,T_r,T_c] int32


def _check_fwd_result(r: FwdResult, q: torch.Tensor, training: bool, masked: bool, need_o: bool = True):
    """Shapes, dtypes, layouts and device of a FwdResult against q (the kernels index τ by
    bh·N + row and the tables by B·H·T_r·T_c: a mismatch would read or write out of bounds)."""
    B, H, N, d = q.shape
    br, bc = block_size(d, q.dtype)
    Tr, Tc = -(-N // br), -(-N // bc)

    def chk(t, shape, dtype, name, contiguous=True):
        if t is None:
            raise ValueError(f"{name} is missing")
        if tuple(t.shape) != shape or t.dtype != dtype or t.device != q.device or (contiguous and not t.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous {dtype} tensor of shape {shape} on {q.device}")

    if need_o:
        if r.o is None or r.o.shape != q.shape or r.o.stride() != q.stride() or r.o.dtype != q.dtype \
                or r.o.device != q.device:
            raise ValueError("o must share q's shape, strides, dtype and device")
    if training:
        chk(r.o2, (B, H, N, d), torch.float32, "o2")
    chk(r.tau, (B, H, N), torch.float32, "tau")
    if masked:
        chk(r.mask, (B, H, Tr, Tc), torch.uint8, "mask")
        chk(r.row_cnt, (B, H, Tr), torch.int32, "row_cnt")
        chk(r.row_idx, (B, H, Tr, Tc), torch.int32, "row_idx")
    elif any(t is not None for t in (r.mask, r.row_cnt, r.row_idx)):
        raise ValueError("unmasked mode: mask, row_cnt and row_idx must all be None")


def entmax_attn_fwd(q, k, v, alpha=1.5, causal=False, n_iter=3, scale=None, training=True,
                    out: FwdResult | None = None, workspace: torch.Tensor | None = None,
                    masked: bool = True) -> FwdResult:
    """Forward pass through the C ABI (see include/entmax_attn.h).  masked=False selects the
    unmasked mode (no block skipping; mask/row_cnt/row_idx are None)."""
    _check_inputs(q, k, v)
    L = _lib.lib()
    s = _shape(q)
    B, H, N, d = q.shape
    br, bc = block_size(d, q.dtype)
    Tr, Tc = -(-N // br), -(-N // bc)
    dev = q.device
    if out is None:
        out = FwdResult(
            # O is written with q's strides (the ABI's "same strides" contract): allocate it so
            o=torch.empty_strided(q.shape, q.stride(), dtype=q.dtype, device=dev),
            o2=torch.empty(q.shape, dtype=torch.float32, device=dev) if training else None,
            tau=torch.empty((B, H, N), dtype=torch.float32, device=dev),
            mask=torch.empty((B, H, Tr, Tc), dtype=torch.uint8, device=dev) if masked else None,
            row_cnt=torch.empty((B, H, Tr), dtype=torch.int32, device=dev) if masked else None,
            row_idx=torch.empty((B, H, Tr, Tc), dtype=torch.int32, device=dev) if masked else None)
    else:
        _check_fwd_result(out, q, training, masked)
    ws_bytes = L.entmax_attn_fwd_workspace_bytes(ctypes.byref(s), _DT[q.dtype], int(causal))
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    st = L.entmax_attn_fwd(_ptr(q), _ptr(k), _ptr(v), ctypes.byref(s), _DT[q.dtype], float(alpha),
                           int(causal), int(n_iter), float(scale or 0.0),
                           _ptr(out.o), _ptr(out.o2), _ptr(out.tau), _ptr(out.mask), _ptr(out.row_cnt),
                           _ptr(out.row_idx), _ptr(workspace), ws_bytes, _stream(dev))
    _lib.check(st, "entmax_attn_fwd")
    return out


def entmax_attn_bwd(q, k, v, d_o, fwd: FwdResult, alpha=1.5, causal=False, scale=None,
                    grads=None, workspace: torch.Tensor | None = None):
    """Backward pass through the C ABI; returns (dq, dk, dv)."""
    if fwd.o2 is None:
        raise ValueError("backward needs O⁽²⁾: run the forward with training=True")
    if d_o.stride() != q.stride() and d_o.shape == q.shape:   # the ABI reads dO with q's strides
        d_o = torch.empty_strided(q.shape, q.stride(), dtype=d_o.dtype, device=d_o.device).copy_(d_o)
    _check_inputs(q, k, v, d_o)
    _check_fwd_result(fwd, q, True, fwd.mask is not None, need_o=False)
    L = _lib.lib()
    s = _shape(q)
    if grads is None:   # written with q's strides (ABI contract), whatever the inputs' layout
        grads = tuple(torch.empty_strided(q.shape, q.stride(), dtype=q.dtype, device=q.device) for _ in range(3))
    for g in grads:
        if g.shape != q.shape or g.stride() != q.stride() or g.dtype != q.dtype or g.device != q.device:
            raise ValueError("grads must share q's shape, strides, dtype and device")
    dq, dk, dv = grads
    ws_bytes = L.entmax_attn_bwd_workspace_bytes(ctypes.byref(s), _DT[q.dtype], int(causal))
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=q.device)
    st = L.entmax_attn_bwd(_ptr(q), _ptr(k), _ptr(v), _ptr(fwd.o2), _ptr(d_o), _ptr(fwd.tau), _ptr(fwd.mask),
                           _ptr(fwd.row_cnt), _ptr(fwd.row_idx), ctypes.byref(s), _DT[q.dtype], float(alpha),
                           int(causal), float(scale or 0.0), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(workspace),
                           ws_bytes, _stream(q.device))
    _lib.check(st, "entmax_attn_bwd")
    return dq, dk, dv


class _EntmaxAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, alpha, causal, n_iter, scale, masked):
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        fw = entmax_attn_fwd(q, k, v, alpha, causal, n_iter, scale, training=True, masked=masked)
        ctx.save_for_backward(q, k, v, fw.o2, fw.tau, fw.mask, fw.row_cnt, fw.row_idx)
        ctx.cfg = (alpha, causal, scale)
        return fw.o

    @staticmethod
    def backward(ctx, d_o):
        q, k, v, o2, tau, mask, row_cnt, row_idx = ctx.saved_tensors
        alpha, causal, scale = ctx.cfg
        fw = FwdResult(None, o2, tau, mask, row_cnt, row_idx)
        dq, dk, dv = entmax_attn_bwd(q, k, v, d_o.contiguous(), fw, alpha, causal, scale)
        return dq, dk, dv, None, None, None, None, None


def entmax_attention(q, k, v, alpha=1.5, causal=False, n_iter=3, scale=None, masked=True):
    """α-entmax attention O = entmax_α(QKᵀ/√d) V with AdaSplash block skipping (autograd op);
    masked=False: the paper's unmasked variant (every visible block, no mask/tables stored)."""
    return _EntmaxAttention.apply(q, k, v, alpha, causal, n_iter, scale, masked)


def profile_enable(on: bool = True):
    _lib.lib().entmax_attn_profile_enable(int(on))


def profile_reset():
    _lib.lib().entmax_attn_profile_reset()


def profile_collect():
    """{kernel name: (launches, total_ms)} since the last reset (synchronises the events)."""
    cap = 64
    names = (ctypes.c_char_p * cap)()
    launches = (ctypes.c_int32 * cap)()
    ms = (ctypes.c_double * cap)()
    n = _lib.lib().entmax_attn_profile_collect(names, launches, ms, cap)
    return {names[i].decode(): (launches[i], ms[i]) for i in range(n)}


# ------------------------------------------------------------------------------------------
# Standalone row-wise α-entmax (include/entmax_rowwise.h)
# ------------------------------------------------------------------------------------------

def _rows_view(x: torch.Tensor):
    if not x.is_cuda:
        raise RuntimeError("entmax_rowwise: tensors must be CUDA tensors (no CPU fallback)")
    if x.dtype not in _DT:
        raise TypeError(f"unsupported dtype {x.dtype}")
    if x.dim() < 1 or x.stride(-1) != 1:
        raise ValueError("last dimension must be contiguous")
    n = x.shape[-1]
    x2 = x.reshape(-1, n)
    if x2.stride(-1) != 1:
        x2 = x2.contiguous()
    return x2, x2.shape[0], n, x2.stride(0) if x2.shape[0] > 1 else n


def _padded_rows(x2: torch.Tensor, rows: int, n: int):
    """(tensor, ld) with a 16-byte-multiple leading dimension (copies only when needed)."""
    q = 16 // x2.element_size()
    ld = x2.stride(0) if rows > 1 else -(-n // q) * q
    if ld % q == 0 and ld >= n:
        return x2, ld
    ldp = -(-n // q) * q
    buf = torch.zeros((rows, ldp), dtype=x2.dtype, device=x2.device)
    buf[:, :n] = x2
    return buf[:, :n], ldp


def entmax_rowwise_fwd(s: torch.Tensor, alpha=1.5, n_iter=3, halley=True):
    """p = α-entmax(s) over the last dimension by T = n_iter Halley-bisection (Alg. 1) or
    bisection (halley=False) iterations; returns (p, τ) with τ in the pre-scaled convention."""
    s2, rows, n, _ = _rows_view(s)
    s2, ld = _padded_rows(s2, rows, n)
    p = torch.empty((rows, ld), dtype=s.dtype, device=s.device)
    t = torch.empty(rows, dtype=torch.float32, device=s.device)
    st = _lib.lib().entmax_rowwise_fwd(_ptr(s2), rows, n, ld, _DT[s.dtype], float(alpha), int(n_iter),
                                       int(bool(halley)), _ptr(p), _ptr(t), _stream(s.device))
    _lib.check(st, "entmax_rowwise_fwd")
    return p[:, :n].reshape(s.shape), t.reshape(s.shape[:-1])


def entmax_rowwise_bwd(p: torch.Tensor, dp: torch.Tensor, alpha=1.5):
    """ds = u ⊙ dp − (⟨u, dp⟩/‖u‖₁)·u with u = p^{2−α}, over the last dimension."""
    if dp.shape != p.shape or dp.dtype != p.dtype:
        raise ValueError("p and dp must share shape and dtype")
    p2, rows, n, _ = _rows_view(p.contiguous())
    d2 = dp.contiguous().reshape(rows, n)
    p2, ld = _padded_rows(p2, rows, n)
    if ld != n:
        d2, _ = _padded_rows(d2, rows, n)
    ds = torch.empty((rows, ld), dtype=p.dtype, device=p.device)
    st = _lib.lib().entmax_rowwise_bwd(_ptr(p2), _ptr(d2), rows, n, ld, _DT[p.dtype], float(alpha), _ptr(ds),
                                       _stream(p.device))
    _lib.check(st, "entmax_rowwise_bwd")
    return ds[:, :n].reshape(p.shape)


class _Entmax(torch.autograd.Function):
    @staticmethod
    def forward(ctx, s, alpha, n_iter, halley):
        p, _ = entmax_rowwise_fwd(s.contiguous(), alpha, n_iter, halley)
        ctx.save_for_backward(p)
        ctx.alpha = alpha
        return p

    @staticmethod
    def backward(ctx, dp):
        (p,) = ctx.saved_tensors
        return entmax_rowwise_bwd(p, dp.contiguous(), ctx.alpha), None, None, None


def entmax(s, alpha=1.5, n_iter=3, halley=True):
    """α-entmax over the last dimension (Eq. 2) by Halley-bisection (autograd op)."""
    return _Entmax.apply(s, alpha, n_iter, halley)


def pack_mask(mask: torch.Tensor) -> torch.Tensor:
    """Bit-packed block mask [..., T_r, ⌈T_c/32⌉] int32 (bit b of word w = M[..., 32w + b])."""
    if not mask.is_cuda or mask.dtype != torch.uint8:
        raise ValueError("mask must be a CUDA uint8 tensor")
    m = mask.contiguous()
    Tc = m.shape[-1]
    rows = m.numel() // Tc
    out = torch.empty(m.shape[:-1] + (-(-Tc // 32),), dtype=torch.int32, device=m.device)
    _lib.check(_lib.lib().entmax_attn_pack_mask(_ptr(m), rows, Tc, _ptr(out), _stream(m.device)),
               "entmax_attn_pack_mask")
    return out
