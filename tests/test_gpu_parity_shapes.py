"""Oracle parity at the benchmarked shapes.

The kernels the bench lines time run here at their own configuration --
V = 64,000 with H = 1,024 / 2,048 (8 N-tiles of 256 in every H-wide GEMM,
the persistent recurrence at full width) and the 1,024-stream scorer -- and
are compared with the C oracle (oracle/desklm_oracle.c, pinned bit-exact to
the compiled reference), never with another GPU path:

* fp32 mode, one window: loss, h_final, dW_in, dW_rec, dW_out and the
  rmsprop step within 1e-4 relative (+ 1e-4 x max-abs floor for
  near-cancelling sums), backprop.hpp:76-222, rmsprop.hpp:113-133;
* bf16 mode, one training window through dl_train_window at the C3 shape
  (and at the C4 width, H = 4,096): the fused dW_out + dense rmsprop
  epilogue (per-row sums of squares over all eight / sixteen N-tiles of an
  M block) against the oracle's rmsprop_update applied to
  the same device gradient (m_out 1e-6 relative, W_out within a few ulps of
  the step), the other updates <= 1 ulp, and the bf16 gradients against the
  fp32 oracle's;
* the persistent bf16 recurrence at H = 2,048, step by step, against a
  float64 evaluation of h' = act(bf16(h) . bf16(W_rec)^T + W_in[x]);
* the C5 scorer (S = 1,024 streams, H = 2,048, V = 64,000): per-token
  log-probabilities of sampled streams against the oracle's
  sharded_logprobs (eval.hpp:151-222), fp32 1e-4, bf16 by its rounding.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RHO, EPS = 0.9995, 1e-6


def close(a, b, rel=1e-4, floor_frac=1e-4):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = max(np.max(np.abs(b)), 1e-30)
    err = np.abs(a - b)
    tol = rel * np.abs(b) + floor_frac * scale
    return bool(np.all(err <= tol)), float(np.max(err / (np.abs(b) + floor_frac * scale)))


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float32."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def make_params(V, H, seed):
    rng = np.random.default_rng(seed)
    return tuple(rng.uniform(-0.1, 0.1, s).astype(np.float32) for s in ((V, H), (H, H), (V, H)))


def make_window(rng, T, B, V, mask_p=0.1):
    x = rng.integers(0, V, (T, B)).astype(np.uint32)
    y = rng.integers(0, V - 1, (T, B)).astype(np.uint32)
    y[y >= 1] += 1  # never bos
    w = (rng.random((T, B)) >= mask_p).astype(np.uint8)
    return x, y, w


def sparse_rows(g_in_dense):
    """Dense W_in gradient -> SparseRowGrads (words, rows) for the oracle's
    rmsprop (row order does not matter to the per-row update)."""
    words = np.flatnonzero(np.any(g_in_dense != 0, axis=1)).astype(np.uint32)
    return words, np.ascontiguousarray(g_in_dense[words])


@pytest.mark.parametrize("precision", ["fp32", "tf32x3"])
@pytest.mark.parametrize("H", [1024, 2048])
def test_fp32_window_and_update_at_c2_c3(orc, H, precision):
    import paper_1502_00512_b200 as dl
    V, T, B = 64000, 4, 8
    rng = np.random.default_rng(H)
    params = make_params(V, H, 100 + H)
    x, y, w = make_window(rng, T, B, V)
    h0 = rng.uniform(0.0, 1.0, (B, H)).astype(np.float32)
    scale, clip, eta = 1.0 / (T * B), 1.0, 0.05
    want = orc.bptt(params, 0, x, y, w, h0, scale, clip)
    m = dl.GpuRnn(V, H, 0, precision)
    m.set_params(*params)
    m.set_opt(None, None, None, RHO, EPS)
    res, hf = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, scale, clip)
    assert res.positions == want["positions"]
    assert res.loss == pytest.approx(want["loss"], rel=1e-4)
    ok, e = close(hf, want["h_final"], floor_frac=1e-5)
    assert ok, ("h_final", e)
    g_in, g_rec, g_out = m.grads()
    for name, got, ref_ in (("dW_in", g_in, want["g_in_dense"]), ("dW_rec", g_rec, want["g_rec"]),
                            ("dW_out", g_out, want["g_out"])):
        ok, e = close(got, ref_)
        assert ok, (name, e)
    # one rmsprop_update on both sides (per-word W_in / W_out scalars)
    assert dl.rmsprop_update(m, eta)
    zero = (np.zeros((H, H), np.float32), np.zeros(V, np.float32), np.zeros(V, np.float32))
    p2, s2, applied = orc.rmsprop(params, zero, want, RHO, EPS, eta)
    assert applied
    for name, got, ref_ in zip(("W_in", "W_rec", "W_out", "m_rec", "m_in", "m_out"),
                               m.params() + m.opt(), p2 + s2):
        ok, e = close(got, ref_)
        assert ok, (name, e)


@pytest.mark.parametrize("V,H", [(64000, 2048), (16384, 4096)])
def test_bf16_fused_window_update_at_c3(orc, V, H):
    """dl_train_window in bf16 mode at V=64,000, H=2,048: the dW_out GEMM
    with the dense W_out rmsprop fused into its epilogue (72 CTA pairs, eight
    N-tiles per 256-row block exchanging per-row sums of squares); and at the
    C4 width H = 4,096 (64 pairs, sixteen N-tiles per block, the persistent
    recurrence at H = 4,096) on a 16,384-word vocabulary."""
    import paper_1502_00512_b200 as dl
    T, B = 4, 64  # TB = 256: the dh / logits GEMMs on pair tiles
    rng = np.random.default_rng(3)
    params = make_params(V, H, 33)
    x, y, w = make_window(rng, T, B, V)
    wb = dl.WindowBatch(x, y, w)
    h0 = rng.uniform(0.0, 1.0, (B, H)).astype(np.float32)
    scale, clip, eta = 1.0 / (T * B), 1.0, 0.01
    # (1) the device's own clipped fp32 dW_out: the unfused GEMM with the
    # same tiles and k order (DL_G16=0 keeps it in fp32)
    os.environ["DL_G16"] = "0"
    try:
        m1 = dl.GpuRnn(V, H, 0, "bf16")
    finally:
        del os.environ["DL_G16"]
    m1.set_params(*params)
    r1, hf1 = dl.bptt_run(m1, wb, h0, scale, clip)
    g_in, g_rec, g_out = m1.grads()
    m1.close()
    # (2) the fused training window
    m2 = dl.GpuRnn(V, H, 0, "bf16")
    m2.set_params(*params)
    m2.set_opt(None, None, None, RHO, EPS)
    r2, hf2, applied = dl.train_window(m2, wb, h0, scale, clip, eta)
    assert applied
    assert r2.loss == r1.loss and r2.positions == r1.positions
    assert np.array_equal(hf2, hf1)
    # (3) the oracle's rmsprop_update (rmsprop.hpp:94-133) on that gradient
    words, rows = sparse_rows(g_in)
    grads = dict(g_in_words=words, g_in_rows=rows, g_rec=g_rec, g_out=g_out)
    zero = (np.zeros((H, H), np.float32), np.zeros(V, np.float32), np.zeros(V, np.float32))
    (w_in2, w_rec2, w_out2), (m_rec2, m_in2, m_out2), ok = orc.rmsprop(params, zero, grads, RHO,
                                                                       EPS, eta)
    assert ok
    gw_in, gw_rec, gw_out = m2.params()
    gm_rec, gm_in, gm_out = m2.opt()
    # m_out: fp64 row sums of the clipped fp32 gradient over all 2,048 columns
    # (partials per 32 columns) vs the reference's sequential double sum
    assert np.allclose(gm_out, m_out2, rtol=1e-6, atol=0), np.max(np.abs(gm_out - m_out2) / m_out2)
    # W_out: w -= float(eta / sqrt(m + eps)) * g in fp32 (the reference rounds
    # eta * g / sqrt(m + eps) once): a few ulps of the step, one of w
    step = (w_out2.astype(np.float64) - params[2])
    tol = 4 * np.spacing(np.abs(step).astype(np.float32)) + np.spacing(np.abs(w_out2))
    err = np.abs(gw_out.astype(np.float64) - w_out2)
    assert np.all(err <= tol), float(np.max(err / tol))
    assert np.mean(np.abs(step) > 0) > 0.99  # the update touched every row
    # W_rec / W_in and their accumulators: the exact kernels, <= 1 ulp
    for name, got, want in (("W_in", gw_in, w_in2), ("W_rec", gw_rec, w_rec2),
                            ("m_rec", gm_rec, m_rec2), ("m_in", gm_in, m_in2)):
        ulps = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
        assert ulps.max() <= 1, (name, ulps.max())
    m2.close()
    # (4) the bf16 window against the fp32 oracle (bf16 operand rounding only)
    want = orc.bptt(params, 0, x, y, w, h0, scale, clip)
    assert r1.positions == want["positions"]
    assert r1.loss == pytest.approx(want["loss"], rel=2e-3)
    assert np.max(np.abs(hf1 - want["h_final"])) < 1e-2
    assert rel_l2(hf1, want["h_final"]) < 2e-3
    for name, got, ref_ in (("dW_out", g_out, want["g_out"]), ("dW_rec", g_rec, want["g_rec"]),
                            ("dW_in", g_in, want["g_in_dense"])):
        assert rel_l2(got, ref_) < 2e-2, (name, rel_l2(got, ref_))


def test_bf16_ds_in_dh_gemm_equals_softmax_kernel():
    """dS formed on the fly in the dh GEMM's operand path (GemmDesc::xf, the
    logits never rewritten in HBM) is bit-identical to the in-place softmax
    rows kernel (DL_XF=0): same loss, h_final, updated parameters and
    accumulators after a training window at the C3 shape (TB = 512)."""
    import paper_1502_00512_b200 as dl
    V, H, T, B = 64000, 2048, 4, 128
    rng = np.random.default_rng(8)
    params = make_params(V, H, 81)
    x, y, w = make_window(rng, T, B, V, mask_p=0.15)
    h0 = rng.uniform(0.0, 1.0, (B, H)).astype(np.float32)
    out = []
    for xf in ("0", "1"):
        os.environ["DL_XF"] = xf
        os.environ["DL_PFAC"] = "0"  # (the in-place kernel, not the shifted exponentials)
        try:
            m = dl.GpuRnn(V, H, 0, "bf16")
        finally:
            del os.environ["DL_XF"]
            del os.environ["DL_PFAC"]
        m.set_params(*params)
        m.set_opt(None, None, None, RHO, EPS)
        r, hf, ok = dl.train_window(m, dl.WindowBatch(x, y, w), h0, 1.0 / (T * B), 1.0, 0.01)
        assert ok
        out.append((r.loss, r.positions, hf, m.params(), m.opt()))
        m.close()
    (l0, p0, h0_, pa, oa), (l1, p1, h1_, pb, ob) = out
    assert l0 == l1 and p0 == p1 and np.array_equal(h0_, h1_)
    for a, b in zip(pa + oa, pb + ob):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("act", [0, 1])
def test_bf16_persistent_recurrence_steps_at_h2048(act):
    """The persistent cluster recurrence (rec_tc.cu) at H = 2,048, B = 128:
    each step's h against float64 act(bf16(h_t) . bf16(W_rec)^T + W_in[x_t])
    computed from the device's own previous state (backprop.hpp:102-112)."""
    import paper_1502_00512_b200 as dl
    V, H, B, T = 4096, 2048, 128, 4
    rng = np.random.default_rng(11 + act)
    w_in, w_rec, w_out = make_params(V, H, 44 + act)
    w_rec = (w_rec * 0.5).astype(np.float32)
    m = dl.GpuRnn(V, H, act, "bf16")
    m.set_params(w_in, w_rec, w_out)
    x = rng.integers(0, V, (T, B)).astype(np.uint32)
    y = rng.integers(2, V, (T, B)).astype(np.uint32)
    w = np.ones((T, B), np.uint8)
    h = rng.uniform(-0.5, 1.0, (B, H)).astype(np.float32)
    Wb = bf16(w_rec).astype(np.float64)
    f = (lambda z: 1.0 / (1.0 + np.exp(-z))) if act == 0 else np.tanh
    h_dev = h
    for t in range(1, T + 1):
        # windows of t steps from the same h0: the first t-1 steps are the
        # same computation, so step t starts from the device's h_{t-1}
        _, hf = dl.bptt_run(m, dl.WindowBatch(x[:t], y[:t], w[:t]), h, 1.0, 1.0,
                            compute_grads=False)
        pre = bf16(h_dev).astype(np.float64) @ Wb.T + w_in[x[t - 1]].astype(np.float64)
        want = f(pre)
        err = np.abs(hf.astype(np.float64) - want)
        assert err.max() < 2e-5, (t, err.max())
        h_dev = hf


@pytest.mark.parametrize("precision", ["fp32", "tf32x3", "bf16"])
def test_c5_scorer_1024_streams(orc, precision):
    """sharded_perplexity's lock-step walk at the C5 shape: 1,024 slices of a
    stream, 3 scoring steps each; 24 slices re-scored by the oracle."""
    import paper_1502_00512_b200 as dl
    V, H, S, n_per = 64000, 2048, 1024, 4
    params = make_params(V, H, 55)
    ids = orc.random_stream(5001, V, S * n_per + 16)[: S * n_per]
    m = dl.GpuRnn(V, H, 0, precision)
    m.set_params(*params)
    # the device scorer over all 1,024 slices (eval.hpp:160-195 layout)
    steps = n_per - 1
    sl = ids.reshape(S, n_per)
    x = np.ascontiguousarray(sl[:, :steps].T)
    t = sl[:, 1:].T.astype(np.int64)
    t[t == 1] = -1
    lp, tot, pred, _ = dl.score(m, x, t)
    r = dl.sharded_perplexity(m, ids, S)
    assert r.predicted == pred and r.total_logprob == pytest.approx(tot, rel=1e-12)
    # oracle: 24 of the slices (first, middle, last), walked the same way
    pick = np.r_[0:8, 508:516, 1016:1024]
    want = orc.sharded_logprobs(params, 0, sl[pick].ravel(), len(pick))
    got = lp[:, pick]
    assert want.shape == got.shape
    mask = ~np.isnan(want)
    assert np.array_equal(mask, ~np.isnan(got))
    if precision != "bf16":
        assert np.allclose(got[mask], want[mask], rtol=1e-4, atol=1e-5)
    else:
        d = np.abs(got[mask] - want[mask])
        assert d.max() < 5e-2 and d.mean() < 1e-2, (d.max(), d.mean())
