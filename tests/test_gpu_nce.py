"""GPU parity of the NCE window (LossMode::kNce, backprop.hpp:126-156 and
193-222; nce.hpp) and its sparse-W_out rmsprop step (rmsprop.hpp:77-92)
against the C oracle, through the C ABI.

The noise draws are the reference's (host mt19937_64 + AliasSampler), so the
generator state after a window must match the oracle's exactly; scores use
the reference's 8-lane double dot product, so losses, gradients and updates
agree to fp32 summation order (1e-4 relative, as the softmax window).
"""
import glob
import os

import numpy as np
import pytest

from test_gpu_window import close, rand_window

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def nce_model(dl, params, counts, k, floor, precision, act=0, seed=5):
    V, H = params[0].shape
    m = dl.GpuRnn(V, H, act, precision)
    m.set_params(*params)
    m.set_loss_mode(0)
    m.set_noise(counts, k, floor)
    m.set_rng_state(dl.rng_seed_state(seed))
    return m


CASES = [
    # V, H, T, B, k, act, mask, clip, floor
    (60, 12, 5, 4, 5, 0, 0.15, 1.0, 1e-3),
    (400, 32, 6, 8, 16, 1, 0.1, 0.5, 1e-8),
    (2000, 128, 8, 16, 64, 0, 0.1, 1.0, 1e-8),
]


@pytest.mark.parametrize("V,H,T,B,k,act,mask,clip,floor", CASES)
def test_nce_window_fp32_matches_oracle(orc, V, H, T, B, k, act, mask, clip, floor):
    import paper_1502_00512_b200 as dl
    rng = np.random.default_rng(V + k)
    params = orc.init_uniform(V, H, 3)
    counts = rng.integers(0, 50, V).astype(np.float64)
    counts[1] = 0
    x, y, w = rand_window(rng, T, B, V, mask)
    h0 = rng.uniform(-0.5, 0.5, (B, H)).astype(np.float32)
    scale = 1.0 / (T * B)
    noise = orc.noise_build(counts, k, floor)
    st = orc.mt_state(5)
    want = orc.bptt_nce(params, act, x, y, w, h0, scale, clip, noise, st)
    m = nce_model(dl, params, counts, k, floor, "fp32", act)
    res, hf = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, scale, clip)
    # the draws consumed exactly the reference's stream
    assert np.array_equal(m.rng_state(), st)
    assert res.positions == want["positions"]
    assert res.loss == pytest.approx(want["loss"], rel=1e-9)
    ok, err = close(hf, want["h_final"])
    assert ok, err
    g_in, g_rec, g_out = m.grads()
    for got, key in ((g_in, "g_in_dense"), (g_rec, "g_rec"), (g_out, "g_out")):
        ok, err = close(got, want[key])
        assert ok, (key, err)
    # the sparse W_out rmsprop step (rmsprop.hpp:77-92) given the gradients
    state = tuple(np.zeros(s, np.float32) for s in ((H, H), V, V))
    p2, s2, ok = orc.rmsprop(params, state, want, 0.9995, 1e-6, 0.05, out_dense=False)
    assert dl.rmsprop_update(m, 0.05)
    for a, b in zip(m.params() + m.opt(), p2 + s2):
        ok, err = close(a, b, rel=1e-4, floor_frac=1e-5)
        assert ok, err
    # untouched W_out rows do not move; their accumulators decay
    touched = np.zeros(V, bool)
    touched[want["g_out_words"]] = True
    assert np.array_equal(m.params()[2][~touched], params[2][~touched])


def test_nce_window_sequence_rng_continues(orc):
    """Consecutive windows keep drawing from the same generator (the
    trainer's rng): after three windows the state equals the oracle's."""
    import paper_1502_00512_b200 as dl
    V, H, T, B, k = 300, 24, 4, 6, 8
    rng = np.random.default_rng(1)
    params = orc.init_uniform(V, H, 9)
    counts = rng.integers(1, 20, V).astype(np.float64)
    noise = orc.noise_build(counts, k, 1e-8)
    st = orc.mt_state(42)
    m = nce_model(dl, params, counts, k, 1e-8, "fp32", seed=42)
    for i in range(3):
        x, y, w = rand_window(rng, T, B, V, 0.2)
        h0 = np.zeros((B, H), np.float32)
        want = orc.bptt_nce(params, 0, x, y, w, h0, 0.1, 1.0, noise, st, compute_grads=False)
        res, _ = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, 0.1, 1.0, compute_grads=False)
        assert res.loss == pytest.approx(want["loss"], rel=1e-9)
        assert np.array_equal(m.rng_state(), st)


def test_nce_window_predrawn_noise_across_shapes_and_reseed(orc):
    """dl_window draws the next window's noise while the device runs the
    current one (runtime.cu nce_predraw): windows that grow past the queue,
    shrink below it, train (bptt + rmsprop) or reseed the generator in
    between all consume exactly the reference's stream."""
    import paper_1502_00512_b200 as dl
    V, H, B, k = 300, 24, 6, 8
    rng = np.random.default_rng(3)
    params = orc.init_uniform(V, H, 9)
    counts = rng.integers(1, 20, V).astype(np.float64)
    noise = orc.noise_build(counts, k, 1e-8)
    st = orc.mt_state(42)
    m = nce_model(dl, params, counts, k, 1e-8, "fp32", seed=42)
    for i, T in enumerate((4, 4, 6, 3, 3, -7, 4, 4)):
        if T < 0:  # reseed: the queue drawn from the old state is dropped
            st = orc.mt_state(-T)
            m.set_rng_state(dl.rng_seed_state(-T))
            continue
        x, y, w = rand_window(rng, T, B, V, 0.2 if i % 2 else 0.0)
        h0 = np.zeros((B, H), np.float32)
        want = orc.bptt_nce(m.params(), 0, x, y, w, h0, 0.1, 1.0, noise, st,
                            compute_grads=False)
        if i == 6:
            res, _, _ = dl.train_window(m, dl.WindowBatch(x, y, w), h0, 0.1, 1.0, 0.01)
        else:
            res, _ = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, 0.1, 1.0, compute_grads=False)
        assert res.loss == pytest.approx(want["loss"], rel=1e-6), i
        assert np.array_equal(m.rng_state(), st), i


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "nce_*.npz"))))
def test_nce_window_matches_reference_fixture(path):
    """Against the reference's own NCE window (tests/golden, made by
    oracle/_ref): loss, rng state after the draws, gradients."""
    import paper_1502_00512_b200 as dl
    g = np.load(path)
    params = (g["w_in"], g["w_rec"], g["w_out"])
    V, H = params[0].shape
    T, B = g["x"].shape
    m = dl.GpuRnn(V, H, 0, "fp32")
    m.set_params(*params)
    m.set_loss_mode(0)
    m.set_noise(g["counts"], int(g["k"]), float(g["floor"]))
    m.set_rng_state(g["rng0"])
    res, hf = dl.bptt_run(m, dl.WindowBatch(g["x"], g["y"], g["w"]), g["h0"], 1.0 / (T * B), 1.0)
    assert np.array_equal(m.rng_state(), g["rng1"])
    assert res.positions == int(g["positions"])
    assert res.loss == pytest.approx(float(g["loss"]), rel=1e-9)
    g_out = np.zeros((V, H), np.float32)
    g_out[g["g_out_words"]] = g["g_out_rows"]
    _, g_rec, got_out = m.grads()
    assert close(g_rec, g["g_rec"])[0]
    assert close(got_out, g_out)[0]


def test_nce_window_bf16_close_to_oracle(orc):
    import paper_1502_00512_b200 as dl
    V, H, T, B, k = 4096, 256, 8, 32, 32
    rng = np.random.default_rng(3)
    params = orc.init_uniform(V, H, 4)
    counts = rng.integers(0, 100, V).astype(np.float64)
    x, y, w = rand_window(rng, T, B, V, 0.1)
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    noise = orc.noise_build(counts, k, 1e-8)
    st = orc.mt_state(5)
    want = orc.bptt_nce(params, 0, x, y, w, h0, 1.0 / (T * B), 1.0, noise, st)
    m = nce_model(dl, params, counts, k, 1e-8, "bf16")
    res, hf = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, 1.0 / (T * B), 1.0)
    assert np.array_equal(m.rng_state(), st)
    assert res.loss == pytest.approx(want["loss"], rel=1e-2)
    _, _, g_out = m.grads()
    cos = float(np.dot(g_out.ravel(), want["g_out"].ravel()) /
                (np.linalg.norm(g_out) * np.linalg.norm(want["g_out"]) + 1e-30))
    assert cos > 0.99
    res2, hf2, ok = dl.train_window(m, dl.WindowBatch(x, y, w), h0, 1.0 / (T * B), 1.0, 0.01)
    assert ok and np.isfinite(res2.loss)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_nce_trainer_matches_oracle(orc, precision):
    """Trainer in NCE mode (the reference default, trainer.hpp:53): the
    device epoch loop draws every window's noise from the trainer's
    mt19937_64 exactly as the reference (state after training identical), and
    its epoch logs follow the oracle's (fp32: summation order; bf16: 1%)."""
    import paper_1502_00512_b200 as dl
    V, H = 40, 8 if precision == "fp32" else 64
    tr, va = orc.random_stream_pair(77, V, 616, 150)
    tr = tr[:600]
    params = orc.init_uniform(V, H, 3)
    # (bf16: a gentler step -- NCE on a 40-word vocabulary amplifies the
    # bf16 operand rounding at eta 0.05)
    kw = dict(nstate=H, noffset=2, minibatch=2, unroll=5, max_epochs=3, mode=0,
              eta=0.05 if precision == "fp32" else 0.005,
              nce_k=7, noise_floor=1e-3, divergence_factor=1e9)
    want = orc.train(oracle_cfg(kw), params, tr, va)
    t = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, precision)
    t.train()
    rel = 1e-4 if precision == "fp32" else 2e-2
    assert t.initial_ppl == pytest.approx(want["initial_ppl"], rel=rel)
    assert len(t.logs) == len(want["logs"])
    for a, b in zip(t.logs, want["logs"]):
        assert a.train_loss == pytest.approx(b[1], rel=rel)
        assert a.valid_ppl == pytest.approx(b[2], rel=5 * rel)
    cur, _ = t.model.trainer_state()
    assert np.array_equal(cur, want["cursors"])
    # the generator advanced by exactly the reference's draws (2 outputs per
    # noise sample, backprop.hpp:126-156): the oracle trainer's final state
    assert np.array_equal(t.model.rng_state(), want["rng_state"])
    assert not np.array_equal(t.model.rng_state(), orc.mt_state(kw.get("seed", 1)))
    # and it survives the RTRN round trip (trainer.hpp:283-285, :312-317)
    t2 = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, precision)
    t2.load_checkpoint(t.save_checkpoint())
    assert np.array_equal(t2.model.rng_state(), t.model.rng_state())


def oracle_cfg(kw):
    import oracle
    return oracle.TrainConfig(**kw)
