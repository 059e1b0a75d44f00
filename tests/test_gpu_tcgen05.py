"""Pin the tcgen05 building blocks (descriptors, TMEM layout of the A
operand, TMEM loads/stores, mbarrier commit) with one 128x128x64 kind::tf32
product through the C ABI."""

import ctypes as C

import numpy as np
import pytest

from gpu_util import needs_gpu

pytestmark = [pytest.mark.gpu, needs_gpu]
torch = pytest.importorskip("torch")


def _tf32(x, mode):
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    if mode == "rna":
        u = (u + 0x1000) & 0xFFFFE000
    else:
        u = u & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def _run(A, B, mode):
    from paper_2211_11172_b200 import _native as N
    lib = N.load()
    a = torch.from_numpy(A).cuda()
    b = torch.from_numpy(B).cuda()
    d = torch.zeros((128, 128), dtype=torch.float32, device="cuda")
    N.check(lib.harl_selftest_tcgen05(a.data_ptr(), b.data_ptr(), d.data_ptr(),
                                      mode,
                                      torch.cuda.current_stream().cuda_stream),
            "selftest")
    return d.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("mode", [0, 1])
def test_tf32_mma_matches_reference(mode):
    rng = np.random.default_rng(mode)
    A = _tf32(rng.standard_normal((128, 64)), "rna").astype(np.float32)
    B = _tf32(rng.standard_normal((64, 128)), "rna").astype(np.float32)
    D = _run(A, B, mode)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    err = np.abs(D - ref).max() / np.abs(ref).max()
    assert err < 1e-5, err


def test_tf32_input_rounding_behaviour():
    """Unrounded fp32 operands: report whether the tensor core truncates or
    rounds (the MLP kernels pre-round both halves, so either is safe)."""
    rng = np.random.default_rng(7)
    A = rng.standard_normal((128, 64)).astype(np.float32)
    B = rng.standard_normal((64, 128)).astype(np.float32)
    D = _run(A, B, 0)
    e_tr = np.abs(D - _tf32(A, "tr") @ _tf32(B, "tr")).max()
    e_rn = np.abs(D - _tf32(A, "rna") @ _tf32(B, "rna")).max()
    print(f"truncate-model err {e_tr:.3e}, round-model err {e_rn:.3e}")
    assert min(e_tr, e_rn) < 1e-3
