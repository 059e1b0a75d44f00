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


@pytest.mark.parametrize("mode", [6, 7])
def test_f16_mma_matches_reference(mode):
    """kind::f16 (fp16 operands, fp32 accumulate): A from TMEM with two
    fp16 per 32-bit column, element k at column k/2, even k in the low half
    (mode 6 -- the operand layout of the 3xFP16 MLP kernels), or A from
    shared memory (mode 7); B in the 2-byte K-major core layout."""
    rng = np.random.default_rng(10 + mode)
    A = rng.standard_normal((128, 64)).astype(np.float16).astype(np.float32)
    B = rng.standard_normal((64, 128)).astype(np.float16).astype(np.float32)
    D = _run(A, B, mode)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    err = np.abs(D - ref).max() / np.abs(ref).max()
    if err > 1e-5 and mode == 6:
        Asw = A.reshape(128, 32, 2)[:, :, ::-1].reshape(128, 64)
        alt = np.abs(D - Asw.astype(np.float64) @ B).max() / np.abs(ref).max()
        pytest.fail(f"err {err:.3e}; with swapped halves {alt:.3e}")
    assert err < 1e-6, err


def test_f16_accumulation_is_fp32():
    """3xFP16 relies on fp32 accumulation of exact fp16 products: a sum of
    small terms onto a large one must keep fp32 (not fp16/tf32) precision."""
    A = np.zeros((128, 64), np.float32)
    B = np.zeros((64, 128), np.float32)
    A[:, 0] = 1.0
    B[0, :] = 1024.0
    A[:, 1:] = 2.0 ** -10
    B[1:, :] = 2.0 ** -4          # 63 products of 2^-14 each
    D = _run(A, B, 6)
    ref = 1024.0 + 63 * 2.0 ** -14
    assert np.all(np.abs(D - ref) <= 2.0 ** -13), (D[0, 0], ref)
