"""Primitive-level B200 check of the tcgen05/TMEM/TMA wrappers (sm100_ptx.cuh, tmap.h)
against torch.matmul, before any attention kernel relies on them."""
import ctypes
import os

import pytest
import torch

pytestmark = pytest.mark.gpu
LIB = os.path.join(os.path.dirname(__file__), "probe", "libprobe.so")


def _lib():
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    L = ctypes.CDLL(LIB)
    L.probe_run.restype = ctypes.c_int
    L.probe_run.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_int]
    return L


@pytest.mark.parametrize("K", [64, 128])
def test_ss_mma_kmajor(K):
    L = _lib()
    g = torch.Generator().manual_seed(K)
    A = torch.randn(128, K, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn(128, K, generator=g).to(torch.bfloat16).cuda()
    D = torch.empty(128, 128, dtype=torch.float32, device="cuda")
    assert L.probe_run(0, A.data_ptr(), B.data_ptr(), None, D.data_ptr(), K, 0) == 0
    ref = A.float() @ B.float().T
    torch.testing.assert_close(D, ref, atol=1e-3, rtol=1e-4)


@pytest.mark.parametrize("Nd", [64, 128])
def test_ss_mma_thread_written_a_mnmajor_b(Nd):
    L = _lib()
    g = torch.Generator().manual_seed(Nd)
    P = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
    V = torch.randn(128, Nd, generator=g).to(torch.bfloat16).cuda()
    D = torch.empty(128, Nd, dtype=torch.float32, device="cuda")
    assert L.probe_run(1, None, V.data_ptr(), P.data_ptr(), D.data_ptr(), 0, Nd) == 0
    ref = P.float() @ V.float()
    torch.testing.assert_close(D, ref, atol=1e-3, rtol=1e-4)


@pytest.mark.parametrize("K", [64, 128])
def test_ts_mma_a_in_tmem(K):
    """A operand written to TMEM by threads (tcgen05.st, bf16 pairs per 32-bit column)."""
    L = _lib()
    g = torch.Generator().manual_seed(100 + K)
    A = torch.randn(128, K, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn(128, K, generator=g).to(torch.bfloat16).cuda()
    D = torch.empty(128, 128, dtype=torch.float32, device="cuda")
    assert L.probe_run(2, None, B.data_ptr(), A.data_ptr(), D.data_ptr(), K, 0) == 0
    torch.testing.assert_close(D, A.float() @ B.float().T, atol=1e-3, rtol=1e-4)
