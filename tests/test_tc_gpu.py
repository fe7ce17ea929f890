"""GPU: the tcgen05 + TMA machinery of the bf16 encoder (fp_tc_node.cu) --
TMA-loaded 128B-swizzled bf16 hi / lo planes, UMMA descriptors, the three
split products accumulated in TMEM, tcgen05.ld epilogue -- against a plain
PyTorch fp64 matmul of the same operands (tolerance 1e-5 relative: bf16
split pairs carry ~16 significant bits)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N", [(128, 32), (300, 64), (4096, 32), (1000, 64)])
def test_tc_split_gemm_matches_fp64(M, N):
    import torch
    from paper_2505_23131_b200 import _native as NV
    g = torch.Generator().manual_seed(M + N)
    x = torch.randn(M, 64, generator=g, dtype=torch.float64)
    w = torch.randn(64, N, generator=g, dtype=torch.float64)
    xf = x.float()
    hi = xf.to(torch.bfloat16)
    lo = (xf - hi.float()).to(torch.bfloat16)
    hi, lo, wd = hi.cuda().contiguous(), lo.cuda().contiguous(), w.cuda().contiguous()
    out = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    NV.check(NV.lib().fp_tc_gemm_selftest(NV.ptr(hi), NV.ptr(lo), NV.ptr(wd), ctypes.c_int32(N),
                                          NV.ptr(out), ctypes.c_int32(M), NV.stream_ptr()))
    torch.cuda.synchronize()
    ref = (x @ w).numpy()
    got = out.cpu().double().numpy()
    scale = np.abs(ref).max()
    assert np.isfinite(got).all()
    assert np.abs(got - ref).max() <= 1e-5 * scale, np.abs(got - ref).max() / scale
