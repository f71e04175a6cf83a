"""tcgen05 building blocks (paper_2603_10026_b200/csrc/sm100.cuh) on one CTA:
TMA SWIZZLE_128B tiles -> UMMA smem/instr descriptors -> tcgen05.mma (SS, TS,
MN-major B, kind::f8f6f4) -> TMEM -> tcgen05.ld, against torch fp32 matmul."""
import ctypes
import os

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _probe():
    h = ctypes.CDLL(os.path.join(ROOT, "paper_2603_10026_b200", "librf_probe.so"))
    h.rf_probe_umma.restype = ctypes.c_int
    h.rf_probe_umma.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_int, ctypes.c_int]
    return h


@pytest.mark.parametrize("mode", [0, 1, 2, 4])
@pytest.mark.parametrize("n", [64, 128, 256])
def test_bf16_umma(mode, n):
    import torch

    k = 128
    torch.manual_seed(mode * 1000 + n)
    a = (torch.rand(128, k, device="cuda") * 2 - 1).bfloat16()
    if mode in (1, 4):
        b = (torch.rand(k, n, device="cuda") * 2 - 1).bfloat16()  # [K][N]
        ref = a.float() @ b.float()
    else:
        b = (torch.rand(n, k, device="cuda") * 2 - 1).bfloat16()  # [N][K]
        ref = a.float() @ b.float().t()
    d = torch.zeros(128, n, device="cuda")
    rc = _probe().rf_probe_umma(mode, a.data_ptr(), b.data_ptr(), d.data_ptr(), n, k)
    assert rc == 0
    err = (d - ref).abs().max().item()
    assert err < 1e-3, (mode, n, err)


@pytest.mark.parametrize("n", [128, 256])
def test_e4m3_umma(n):
    import torch

    k = 128
    torch.manual_seed(n)
    a = (torch.rand(128, k, device="cuda") * 8 - 4).to(torch.float8_e4m3fn)
    b = (torch.rand(n, k, device="cuda") * 2 - 1).to(torch.float8_e4m3fn)
    ref = a.float() @ b.float().t()
    d = torch.zeros(128, n, device="cuda")
    rc = _probe().rf_probe_umma(3, a.data_ptr(), b.data_ptr(), d.data_ptr(), n, k)
    assert rc == 0
    assert (d - ref).abs().max().item() < 1e-3
