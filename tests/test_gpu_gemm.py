"""The tcgen05/TMEM/TMA GEMM engine (gemm_tc.cu) and the fp32 SIMT engine
(gemm_simt.cu) against an fp64 numpy product of the same (bf16-rounded)
inputs, for every operand layout the RNNLM window uses, ragged shapes
(V = 10,000 is not a tile multiple), split-K, and the online-LSE logits
epilogue."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bf16_round(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32)


def run_gemm(m, M, N, K, am, bm, A, B, splits=1, tgt=None):
    from paper_1502_00512_b200._lib import check, load
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    if tgt is None:
        out = np.empty(M * N, np.float32)
        tp = None
    else:
        out = np.empty(M * N + 2 * M, np.float32)
        tgt = np.ascontiguousarray(tgt, np.uint32)
        tp = tgt.ctypes.data
    check(load().dl_test_gemm(m.handle, M, N, K, am, bm, A.ctypes.data, B.ctypes.data,
                              out.ctypes.data, splits, tp), m.handle)
    return out


SHAPES = [  # M, N, K
    (128, 128, 64), (128, 256, 128), (256, 512, 192), (64, 128, 128),
    (200, 300, 100), (384, 1000, 136), (128, 2048, 512), (2048, 128, 640),
]


@pytest.mark.parametrize("precision", ["bf16", "fp32", "tf32x3"])
@pytest.mark.parametrize("am,bm", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_layouts(precision, am, bm, M, N, K):
    import paper_1502_00512_b200 as dl
    if precision == "bf16" and (M % 8 or N % 8 or K % 8):
        pytest.skip("TMA needs 16-byte row pitch")
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    if precision == "bf16":
        A, B = bf16_round(A), bf16_round(B)
    want = A.astype(np.float64) @ B.astype(np.float64).T
    m = dl.GpuRnn(8, 8, 0, precision)
    As = A if am == 0 else np.ascontiguousarray(A.T)
    Bs = B if bm == 0 else np.ascontiguousarray(B.T)
    for splits in (1, 3):
        got = run_gemm(m, M, N, K, am, bm, As, Bs, splits).reshape(M, N)
        err = np.abs(got - want).max()
        assert err <= 1e-4 * np.sqrt(K), (splits, err)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 10000, 128), (300, 1000, 256),
                                   (2048, 4096, 1024)])
def test_logits_epilogue(M, N, K):
    import paper_1502_00512_b200 as dl
    rng = np.random.default_rng(N + K)
    A = bf16_round(rng.uniform(-1, 1, (M, K)).astype(np.float32))
    B = bf16_round(rng.uniform(-0.2, 0.2, (N, K)).astype(np.float32))
    tgt = rng.integers(0, N, M).astype(np.uint32)
    S = A.astype(np.float64) @ B.astype(np.float64).T
    mx = S.max(1, keepdims=True)
    lse = (mx + np.log(np.exp(S - mx).sum(1, keepdims=True)))[:, 0]
    want_lp = S[np.arange(M), tgt] - lse
    m = dl.GpuRnn(8, 8, 0, "bf16")
    out = run_gemm(m, M, N, K, 0, 0, A, B, 1, tgt)
    logits = out[: M * N].reshape(M, N)
    lp = out[M * N: M * N + M]
    tl = out[M * N + M:]
    assert np.abs(tl - S[np.arange(M), tgt]).max() < 1e-3
    assert np.abs(logits - S).max() <= np.abs(S).max() * 2 ** -8 + 1e-3
    assert np.abs(lp - want_lp).max() < 2e-3
