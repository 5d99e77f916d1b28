"""tcgen05 building blocks: UMMA descriptors (no swizzle and 128 B swizzle),
TMA tensor-map loads, UMMA issue, commit, TMEM readback."""

import ctypes

import pytest
import torch

from paper_2605_14217_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("K,N", [(64, 16), (64, 32), (512, 16), (512, 32), (128, 256), (256, 128)])
def test_tc_selftest_gemm(cuda_device, mode, K, N):
    g = torch.Generator(device=cuda_device)
    g.manual_seed(K * 1000 + N + mode)
    A = torch.randn(128, K, generator=g, device=cuda_device).to(torch.bfloat16)
    B = torch.randn(N, K, generator=g, device=cuda_device).to(torch.bfloat16)
    D = torch.full((128, N), float("nan"), device=cuda_device)
    s = torch.cuda.current_stream(cuda_device)
    rc = _lib.load().preft_tc_selftest(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                       ctypes.c_void_p(D.data_ptr()), K, N, mode, ctypes.c_void_p(s.cuda_stream))
    _lib.check(rc, "tc_selftest")
    torch.cuda.synchronize()
    ref = A.double() @ B.double().T
    err = (D.double() - ref).abs().max().item()
    assert err <= 1e-4 * ref.abs().max().item() + 1e-5, f"mode {mode}: max err {err}"
