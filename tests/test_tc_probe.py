"""tcgen05 / TMEM / TMA encoding probe (test-only library tests/native/libtcprobe.so):
the descriptor, swizzle and operand-major conventions every tensor-core
kernel in csrc/ relies on, checked against a torch fp32 GEMM."""

import ctypes
import os

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu
LIB = os.path.join(ROOT, "tests", "native", "libtcprobe.so")


@pytest.fixture(scope="module")
def probe():
    L = ctypes.CDLL(LIB)
    L.tc_probe.restype = ctypes.c_int
    L.tc_probe.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int, ctypes.c_int]
    return L


@pytest.mark.parametrize("mode,N", [(0, 256), (0, 16), (1, 256), (1, 16), (1, 64), (2, 128),
                                    (2, 64), (3, 256), (3, 16), (4, 16), (4, 128)])
def test_gemm_encodings(probe, mode, N):
    g = torch.Generator().manual_seed(mode * 1000 + N)
    A = torch.randn(128, 128, generator=g).to(torch.bfloat16).cuda()
    B = torch.randn(N, 128, generator=g).to(torch.bfloat16).cuda()
    Bt = B.t().contiguous()
    D = torch.zeros(128, N, dtype=torch.float32, device="cuda")
    At = A.t().contiguous()
    rc = probe.tc_probe(A.data_ptr(), B.data_ptr(), Bt.data_ptr(), At.data_ptr(), D.data_ptr(), N, mode)
    assert rc == 0
    ref = A.float() @ B.float().t()
    err = (D - ref).abs().max().item()
    assert err < 1e-2 * ref.abs().max().item(), (mode, N, err)
