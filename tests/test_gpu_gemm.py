"""Kernel unit tests for the tcgen05/TMA bf16 GEMM (through the C-ABI test entry), against numpy
fp64 on bf16-representable inputs.  Tolerance: fp32 accumulation of K bf16 products -> normwise
<= 1e-5 (about sqrt(K) 2^-24 relative, with margin)."""
import numpy as np
import pytest

from synth.gen import round_bf16

pytestmark = pytest.mark.gpu


def _mk(shape, seed):
    return round_bf16(np.random.default_rng(seed).standard_normal(shape).astype(np.float32))


def _run(M, N, K, a_mn, b_mn, splits=0, seed=0, reps=1, init=None):
    import torch

    from paper_2004_09910_b200.tgp import test_gemm_bf16

    A = _mk((M, K), seed)          # logical A[m][k]
    Bm = _mk((N, K), seed + 1)     # logical B[n][k]
    ref = A.astype(np.float64) @ Bm.astype(np.float64).T   # D[m][n]
    a_mem = A.T.copy() if a_mn else A
    b_mem = Bm.T.copy() if b_mn else Bm
    dA = torch.tensor(a_mem, device="cuda").to(torch.bfloat16)
    dB = torch.tensor(b_mem, device="cuda").to(torch.bfloat16)
    outs = []
    for _ in range(reps):
        D = torch.full((M * N,), float("nan"), device="cuda") if init is None else \
            torch.tensor(init.ravel(), dtype=torch.float32, device="cuda")
        test_gemm_bf16(dA, dB, D, M, N, K, a_mn, b_mn, splits)
        d = D.cpu().numpy().astype(np.float64)
        d = d.reshape(M, N) if b_mn else d.reshape(N, M).T
        outs.append(d)
    return outs, ref


@pytest.mark.parametrize("M,N,K,a_mn,splits", [
    (128, 16, 64, False, 1), (128, 16, 256, False, 0), (256, 16, 1024, False, 4), (4096, 16, 4096, False, 0),
    (4096, 16, 4096, False, 8), (512, 8, 512, False, 2), (384, 24, 640, False, 0), (1024, 64, 2048, False, 0),
    (512, 128, 512, False, 0), (256, 256, 512, False, 0), (256, 512, 256, False, 0),
    (128, 16, 64, True, 1), (4096, 16, 4096, True, 0), (1024, 32, 1024, True, 4), (256, 200, 512, True, 0),
])
def test_gemm_skinny(M, N, K, a_mn, splits):
    outs, ref = _run(M, N, K, a_mn, False, splits)
    d = outs[0]
    assert np.isfinite(d).all()
    err = np.max(np.abs(d - ref)) / np.max(np.abs(ref))
    assert err <= 1e-5, err


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (256, 256, 512), (4096, 4096, 512), (512, 384, 192), (1024, 2048, 256)])
def test_gemm_wgrad_mn_major(M, N, K):
    outs, ref = _run(M, N, K, True, True)
    d = outs[0]
    assert np.isfinite(d).all()
    err = np.max(np.abs(d - ref)) / np.max(np.abs(ref))
    assert err <= 1e-5, err


def test_gemm_split_k_deterministic():
    # fixed-order DSMEM reduction: repeated runs are bitwise identical (reading Z21)
    outs, ref = _run(2048, 16, 4096, False, False, splits=8, reps=3)
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (4096, 4096, 512), (512, 384, 192), (1024, 2048, 256), (256, 128, 40)])
def test_gemm_dw_persistent(M, N, K):
    # the persistent deferred-dW kernel (W_j): store, then accumulate (TMA reduce-add) into the result
    outs, ref = _run(M, N, K, True, True, splits=-1)
    d = outs[0]
    assert np.isfinite(d).all()
    assert np.max(np.abs(d - ref)) / np.max(np.abs(ref)) <= 1e-5
    init = np.random.default_rng(3).standard_normal((M, N)).astype(np.float32)
    outs2, _ = _run(M, N, K, True, True, splits=-2, init=init)
    assert np.max(np.abs(outs2[0] - (ref + init))) / np.max(np.abs(ref + init)) <= 1e-5
