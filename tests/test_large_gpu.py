"""Maximum sizes: tensors past 2^31 elements (64-bit offsets end to end).

B200 has 180 GB of HBM, so a single f64 tensor can exceed 2^31 elements (17.2 GB). These
tests permute and contract such tensors through the C ABI and check them on the device
against torch (used only as the checker) -- the oracle cannot hold these sizes in seconds.
Skipped when the device has less than the memory they need."""
import numpy as np
import pytest

import paper_2401_01921_b200 as tnb
from paper_2401_01921_b200 import _lib, dense

pytestmark = pytest.mark.gpu

BIG = (1 << 31) + (1 << 22)  # elements: past the 32-bit boundary


def _need(cuda, gbytes):
    import torch
    free, _ = torch.cuda.mem_get_info(cuda)
    if free < gbytes * (1 << 30):
        pytest.skip(f"needs {gbytes} GiB free on the device")


def test_permute_past_2_31_elements(cuda):
    """t2d and row-gather permutes of a 2.15G-element f64 tensor: bit-exact against torch's
    own permute().contiguous() of the same buffer."""
    import torch
    _need(cuda, 56)
    shape = (2049, 1024, 1025)  # 2,150,629,376 elements
    assert int(np.prod(shape)) > (1 << 31)
    src = torch.empty(shape, dtype=torch.float64, device=cuda)
    src.view(-1)[:] = torch.arange(src.numel(), dtype=torch.float64, device=cuda)
    t = dense.DenseTensor(src)
    for perm in ((2, 1, 0), (1, 0, 2)):
        out = t.permute(*perm).contiguous()
        want = src.permute(*perm).contiguous()
        assert torch.equal(out._buf.view(want.shape), want), perm
        del out, want
        torch.cuda.empty_cache()


def test_contract_output_past_2_31_elements(cuda):
    """A GEMM whose output has more than 2^31 elements (strided stores, tile offsets):
    checked on sampled rows against torch's float64 matmul."""
    import torch
    _need(cuda, 24)
    M, K, N = 65536, 24, 32832  # out: 2,151,677,952 elements (17.2 GB)
    assert M * N > (1 << 31)
    g = torch.Generator(device=cuda).manual_seed(0)
    a = torch.randn((M, K), dtype=torch.float64, device=cuda, generator=g)
    b = torch.randn((K, N), dtype=torch.float64, device=cuda, generator=g)
    out = torch.empty((M, N), dtype=torch.float64, device=cuda)
    _lib.contract_dense(a.data_ptr(), _lib.TNB_F64, (M, K), (0, 1), b.data_ptr(), _lib.TNB_F64, (K, N), (0, 1),
                        [1], [0], out.data_ptr(), _lib.CPLX_4M, dense.stream_handle())
    torch.cuda.synchronize()
    rows = torch.tensor([0, 1, 12345, M // 2, M - 2, M - 1], device=cuda)
    want = a[rows] @ b
    got = out[rows]
    err = (got - want).norm() / want.norm()
    assert err.item() <= 1e-13
    # the last row lies beyond element 2^31: it must be written, not left uninitialised
    assert torch.isfinite(out[-1]).all() and (out[-1] - a[-1] @ b).abs().max().item() <= 1e-11
