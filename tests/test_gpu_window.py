"""GPU parity of one truncated-BPTT window (bptt_run softmax mode,
backprop.hpp:76-222) and the rmsprop update (rmsprop.hpp:113-133) against
the C oracle, through the C ABI.

Tolerances (north star): fp32 mode -- loss / h_final / gradients within
1e-4 relative, with an absolute floor of 1e-4 x the matrix max-abs for
near-cancelling gradient sums; rmsprop bit-exact given identical gradients
(<= 1 float ulp where a double sum of squares lands on a rounding tie).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL = 1e-4


def rand_window(rng, T, B, V, mask_p):
    x = rng.integers(0, V, (T, B)).astype(np.uint32)
    y = rng.integers(0, V - 1, (T, B)).astype(np.uint32)
    y[y >= 1] += 1  # never bos (test_backprop.cpp:41-45)
    w = (rng.random((T, B)) >= mask_p).astype(np.uint8)
    return x, y, w


def close(a, b, rel=REL, floor_frac=1e-4):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = max(np.max(np.abs(b)), 1e-30)
    err = np.abs(a - b)
    tol = rel * np.abs(b) + floor_frac * scale
    return bool(np.all(err <= tol)), float(np.max(err / (np.abs(b) + floor_frac * scale)))


CASES = [
    # V, H, T, B, act, mask, clip
    (7, 5, 4, 2, 0, 0.15, 3.4e38),
    (50, 16, 5, 3, 1, 0.2, 0.05),
    (333, 64, 8, 8, 0, 0.1, 1.0),
    (1000, 128, 8, 8, 0, 0.1, 1.0),
    (2048, 256, 4, 32, 1, 0.1, 0.5),
    (10000, 128, 8, 8, 0, 0.1, 1.0),  # C1 shape
]


@pytest.mark.parametrize("precision", ["fp32", "tf32x3"])
@pytest.mark.parametrize("V,H,T,B,act,mask,clip", CASES)
def test_window_fp32_matches_oracle(orc, V, H, T, B, act, mask, clip, precision):
    import paper_1502_00512_b200 as dl
    rng = np.random.default_rng(V * 31 + H)
    params = orc.init_uniform(V, H, 11 + V)
    x, y, w = rand_window(rng, T, B, V, mask)
    h0 = rng.uniform(-0.5, 0.5, (B, H)).astype(np.float32)
    scale = 1.0 / (T * B)
    want = orc.bptt(params, act, x, y, w, h0, scale, clip)
    m = dl.GpuRnn(V, H, act, precision)
    m.set_params(*params)
    res, hf = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, scale, clip)
    assert res.positions == want["positions"]
    assert res.loss == pytest.approx(want["loss"], rel=REL)
    ok, e = close(hf, want["h_final"], floor_frac=1e-5)
    assert ok, e
    g_in, g_rec, g_out = m.grads()
    for got, ref_ in ((g_in, want["g_in_dense"]), (g_rec, want["g_rec"]), (g_out, want["g_out"])):
        ok, e = close(got, ref_)
        assert ok, e
    # clip bounds every component (test_backprop.cpp:489-513)
    for g in (g_in, g_rec, g_out):
        assert np.all(np.abs(g) <= np.float32(min(clip, 3.4e38)))
    # determinism: identical inputs -> bit-identical results (test_backprop.cpp:515-536)
    res2, hf2 = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, scale, clip)
    g2 = m.grads()
    assert res2.loss == res.loss and np.array_equal(hf2, hf)
    for a, b in zip(g2, (g_in, g_rec, g_out)):
        assert np.array_equal(a, b)


def test_masked_window_has_zero_loss_and_grads(orc):
    import paper_1502_00512_b200 as dl
    V, H, T, B = 40, 8, 4, 2
    rng = np.random.default_rng(131)
    params = orc.init_uniform(V, H, 51)
    x, y, _ = rand_window(rng, T, B, V, 0.0)
    w = np.zeros((T, B), np.uint8)
    h0 = rng.uniform(-0.5, 0.5, (B, H)).astype(np.float32)
    m = dl.GpuRnn(V, H, 0, "fp32")
    m.set_params(*params)
    res, _ = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, 1.0, 3.4e38)
    assert res.loss == 0.0 and res.positions == 0
    for g in m.grads():
        assert not np.any(g)


def test_loss_only_window(orc):
    import paper_1502_00512_b200 as dl
    V, H, T, B = 300, 32, 6, 4
    rng = np.random.default_rng(7)
    params = orc.init_uniform(V, H, 5)
    x, y, w = rand_window(rng, T, B, V, 0.2)
    h0 = rng.uniform(-0.5, 0.5, (B, H)).astype(np.float32)
    want = orc.bptt(params, 0, x, y, w, h0, 0.5, 1.0, compute_grads=False)
    m = dl.GpuRnn(V, H, 0, "fp32")
    m.set_params(*params)
    res, hf = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, 0.5, 1.0, compute_grads=False)
    assert res.loss == pytest.approx(want["loss"], rel=REL)
    assert res.positions == want["positions"]


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("V,H", [(64, 32), (304, 512), (200, 2048)])
def test_rmsprop_bitexact_given_identical_grads(orc, precision, V, H):
    """rmsprop_update on injected oracle gradients: W and m bit-exact.  H >=
    512 runs the block-per-row kernel (kernels.cu k_rms_rows_blk) for the
    sparse W_in rows and the dense W_out rows."""
    import paper_1502_00512_b200 as dl
    T, B = 5, 3
    rng = np.random.default_rng(157)
    params = orc.init_uniform(V, H, 97)
    x, y, w = rand_window(rng, T, B, V, 0.1)
    h0 = rng.uniform(-0.5, 0.5, (B, H)).astype(np.float32)
    g = orc.bptt(params, 0, x, y, w, h0, 1.0 / (T * B), 1.0)
    state = (rng.uniform(0, 0.01, (H, H)).astype(np.float32),
             rng.uniform(0, 0.01, V).astype(np.float32),
             rng.uniform(0, 0.01, V).astype(np.float32))
    p2, s2, applied = orc.rmsprop(params, state, g, 0.9995, 1e-6, 0.05)
    m = dl.GpuRnn(V, H, 0, precision)
    m.set_params(*params)
    m.set_opt(*state, 0.9995, 1e-6)
    m.set_grads(g["g_in_words"], g["g_in_rows"], g["g_rec"], g["g_out"])
    assert dl.rmsprop_update(m, 0.05) == applied
    for got, want in zip(m.params() + m.opt(), p2 + s2):
        ulps = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
        assert ulps.max() <= 1, ulps.max()
        assert np.mean(ulps == 0) > 0.999


def test_rmsprop_rejects_nonfinite_untouched(orc):
    """rmsprop.hpp:111-116 (test_backprop.cpp:687-699)."""
    import paper_1502_00512_b200 as dl
    V, H = 5, 3
    params = orc.init_uniform(V, H, 99)
    m = dl.GpuRnn(V, H, 0, "fp32")
    m.set_params(*params)
    m.set_opt(None, None, None, 0.9, 1e-6)
    g_rec = np.zeros((H, H), np.float32)
    g_rec[0, 0] = np.nan
    m.set_grads(np.zeros(0, np.uint32), np.zeros((0, H), np.float32), g_rec,
                np.zeros((V, H), np.float32))
    assert dl.rmsprop_update(m, 0.1) is False
    for a, b in zip(m.params(), params):
        assert np.array_equal(a, b)
    for s in m.opt():
        assert not np.any(s)


def test_rmsprop_hand_computation():
    """test_backprop.cpp:609-639: m = 0.5*8 + 0.5*12.5 = 10.25."""
    import paper_1502_00512_b200 as dl
    m = dl.GpuRnn(4, 2, 0, "fp32")
    z = np.zeros((4, 2), np.float32)
    m.set_params(z, np.zeros((2, 2), np.float32), z)
    m_in = np.zeros(4, np.float32)
    m_in[2] = 8.0
    m.set_opt(None, m_in, None, 0.5, 1e-6)
    g_rec = np.zeros((2, 2), np.float32)
    g_rec[1, 0] = 2.0
    m.set_grads(np.array([2], np.uint32), np.array([[3.0, 4.0]], np.float32), g_rec,
                np.zeros((4, 2), np.float32))
    assert dl.rmsprop_update(m, 0.1)
    w_in, w_rec, _ = m.params()
    m_rec, m_in2, _ = m.opt()
    denom = np.sqrt(10.25 + 1e-6)
    assert m_in2[2] == pytest.approx(10.25, abs=1e-5)
    assert w_in[2, 0] == pytest.approx(-0.1 * 3.0 / denom, abs=1e-6)
    assert w_in[2, 1] == pytest.approx(-0.1 * 4.0 / denom, abs=1e-6)
    assert w_in[0, 0] == 0.0 and m_in2[0] == 0.0
    assert w_rec[1, 0] == pytest.approx(-0.1 * 2.0 / np.sqrt(0.5 * 4.0 + 1e-6), abs=1e-6)
    assert m_rec[1, 0] == pytest.approx(2.0, abs=1e-6)


def test_window_then_update_matches_oracle_step(orc):
    """One full training step (window + rmsprop) in fp32 mode."""
    import paper_1502_00512_b200 as dl
    V, H, T, B = 500, 64, 8, 8
    rng = np.random.default_rng(3)
    params = orc.init_uniform(V, H, 17)
    x, y, w = rand_window(rng, T, B, V, 0.1)
    h0 = np.full((B, H), 0.5, np.float32)
    g = orc.bptt(params, 0, x, y, w, h0, 1.0 / (T * B), 1.0)
    zero = (np.zeros((H, H), np.float32), np.zeros(V, np.float32), np.zeros(V, np.float32))
    p2, s2, _ = orc.rmsprop(params, zero, g, 0.9995, 1e-6, 0.05)
    m = dl.GpuRnn(V, H, 0, "fp32")
    m.set_params(*params)
    dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, 1.0 / (T * B), 1.0)
    assert dl.rmsprop_update(m, 0.05)
    for got, want in zip(m.params(), p2):
        ok, e = close(got, want, rel=1e-4, floor_frac=1e-4)
        assert ok, e


@pytest.mark.parametrize("precision,V,H", [("fp32", 300, 40), ("bf16", 1000, 256),
                                           ("bf16", 4000, 512)])
def test_train_window_equals_window_then_rmsprop(orc, precision, V, H):
    """dl_train_window = dl_window + dl_rmsprop (Trainer::run_epoch's pair,
    trainer.hpp:391-397): identical in fp32; in bf16 the W_out update runs in
    the dW_out epilogue (fp32 step arithmetic), so W_out / m_out agree to
    rounding."""
    import paper_1502_00512_b200 as dl
    rng = np.random.default_rng(V)
    T, B = 6, 64
    params = orc.init_uniform(V, H, 2)
    x = rng.integers(0, V, (T, B)).astype(np.uint32)
    y = rng.integers(2, V, (T, B)).astype(np.uint32)
    w = (rng.random((T, B)) > 0.1).astype(np.uint8)
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    wb = dl.WindowBatch(x, y, w)
    out = []
    for fused_call in (False, True):
        # the separate path with the fp32 dW_out (DL_G16=0), as the fused
        # epilogue updates from the fp32 accumulator
        os.environ["DL_G16"] = "0"
        try:
            m = dl.GpuRnn(V, H, 0, precision)
        finally:
            os.environ.pop("DL_G16", None)
        m.set_params(*params)
        if fused_call:
            res, hf, ok = dl.train_window(m, wb, h0, 1.0 / (T * B), 1.0, 0.05)
        else:
            res, hf = dl.bptt_run(m, wb, h0, 1.0 / (T * B), 1.0)
            ok = dl.rmsprop_update(m, 0.05)
        assert ok
        out.append((res, hf, m.params(), m.opt()))
        m.close()
    (r1, h1, p1, o1), (r2, h2, p2, o2) = out
    assert r1.positions == r2.positions
    assert r1.loss == r2.loss
    assert np.array_equal(h1, h2)
    if precision == "fp32":
        for a, b in zip(p1 + o1, p2 + o2):
            assert np.array_equal(a, b)
    else:
        for a, b in zip(p1, p2):
            np.testing.assert_allclose(a, b, rtol=1e-5, atol=1e-7)
        for a, b in zip(o1, o2):
            np.testing.assert_allclose(a, b, rtol=1e-3, atol=1e-12)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("V,H,T,B,mask", [(8, 8, 1, 1, 0.0), (16, 8, 3, 2, 1.0), (64, 16, 1, 5, 0.5)])
def test_degenerate_windows_match_oracle(orc, precision, V, H, T, B, mask):
    """Edge shapes the reference tests exercise: a single position, a fully
    masked window (no scored positions: zero loss, zero output gradient),
    one step of several streams."""
    import paper_1502_00512_b200 as dl
    rng = np.random.default_rng(V * 7 + T)
    params = orc.init_uniform(V, H, 2)
    x, y, w = rand_window(rng, T, B, V, 0.0)
    if mask == 1.0:
        w[:] = 0
    elif mask > 0.0:
        w[:, ::2] = 0
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    want = orc.bptt(params, 0, x, y, w, h0, 1.0 / (T * B), 1.0)
    m = dl.GpuRnn(V, H, 0, precision)
    m.set_params(*params)
    res, hf = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, 1.0 / (T * B), 1.0)
    assert res.positions == want["positions"]
    tol = 1e-4 if precision == "fp32" else 2e-2
    assert res.loss == pytest.approx(want["loss"], rel=tol, abs=1e-12)
    g_in, g_rec, g_out = m.grads()
    if mask == 1.0:
        assert res.loss == 0.0 and not np.any(g_out) and not np.any(g_rec) and not np.any(g_in)
    else:
        ok, err = close(g_out, want["g_out"], rel=tol, floor_frac=1e-3 if precision == "bf16" else 1e-4)
        assert ok, err
    assert dl.rmsprop_update(m, 0.05)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_v65536_shape_check(orc, precision):
    """V = 65,536 (2^16, tile-aligned everywhere) once as a
    shape check next to the 64,000 / 10,000 configurations."""
    import paper_1502_00512_b200 as dl
    V, H, T, B = 65536, 256, 2, 16
    rng = np.random.default_rng(65536)
    params = orc.init_uniform(V, H, 6)
    x, y, w = rand_window(rng, T, B, V, 0.1)
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    want = orc.bptt(params, 0, x, y, w, h0, 1.0 / (T * B), 1.0)
    m = dl.GpuRnn(V, H, 0, precision)
    m.set_params(*params)
    res, hf = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, 1.0 / (T * B), 1.0)
    tol = 1e-4 if precision == "fp32" else 1e-2
    assert res.positions == want["positions"]
    assert res.loss == pytest.approx(want["loss"], rel=tol)
    g_out = m.grads()[2]
    cos = float(np.dot(g_out.ravel(), want["g_out"].ravel()) /
                (np.linalg.norm(g_out) * np.linalg.norm(want["g_out"]) + 1e-30))
    assert cos > (0.99999 if precision == "fp32" else 0.99)
