"""Pins the C oracle (oracle/desklm_oracle.c) before it is trusted as the GPU
checker: bit-exact against the committed reference fixtures (tests/golden,
made by tests/golden/make_golden.py from the compiled reference), against
the reference itself on randomised configurations when oracle/_ref is
present, and against the reference tests' known-answer values."""
import glob
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name), allow_pickle=False)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "window_*.npz"))))
def test_window_golden_bitexact(orc, path):
    g = load(path)
    params = (g["w_in"], g["w_rec"], g["w_out"])
    r = orc.bptt(params, int(g["act"]), g["x"], g["y"], g["w"], g["h0"],
                 1.0 / (int(g["T"]) * int(g["B"])), float(g["clip"]))
    assert r["loss"] == float(g["loss"])
    assert r["positions"] == int(g["positions"])
    for k in ("h_final", "g_in_words", "g_in_rows", "g_rec", "g_out"):
        assert np.array_equal(r[k], g[k]), k
    state = (g["m_rec"], g["m_in"], g["m_out"])
    p2, s2, applied = orc.rmsprop(params, state, r, 0.9995, 1e-6, 0.05)
    assert applied == bool(g["applied"])
    for a, k in zip(p2 + s2, ("u_w_in", "u_w_rec", "u_w_out", "u_m_rec", "u_m_in", "u_m_out")):
        assert np.array_equal(a, g[k]), k


def test_score_golden_bitexact(orc):
    g = load("score.npz")
    params = (g["w_in"], g["w_rec"], g["w_out"])
    act, shards = int(g["act"]), int(g["shards"])
    lp = orc.sharded_logprobs(params, act, g["ids"], shards)
    assert np.array_equal(np.isnan(lp), np.isnan(g["logprobs"]))
    ok = ~np.isnan(lp)
    assert np.array_equal(lp[ok], g["logprobs"][ok])
    sp = orc.sharded_ppl(params, act, g["ids"], shards)
    assert [sp["total_logprob"], sp["predicted"], sp["perplexity"]] == list(g["sharded"])
    rp = orc.rnn_ppl(params, act, g["ids"])
    assert [rp["total_logprob"], rp["predicted"], rp["perplexity"]] == list(g["rnn"])


def test_train_golden_bitexact(orc):
    """Three softmax epochs of Trainer<StandardTraits>: logs and the final
    parameters/optimiser/cursors/hidden inside the RTRN bytes."""
    from paper_1502_00512_b200 import TrainConfig, formats
    g = load("train.npz")
    params = (g["w_in"], g["w_rec"], g["w_out"])
    cfg = oracle.TrainConfig(nstate=8, noffset=2, minibatch=2, unroll=5, eta=0.05,
                             max_epochs=3, mode=1)
    r = orc.train(cfg, params, g["train"], g["valid"])
    assert r["initial_ppl"] == float(g["initial"])
    assert np.array_equal(r["logs"][:, [0, 1, 2, 3, 6]], g["logs"][:, [0, 1, 2, 3, 6]])
    pcfg = TrainConfig(nstate=8, noffset=2, minibatch=2, unroll=5, eta=0.05, max_epochs=3,
                       mode=1)
    st = formats.read_trainer(g["rtrn"].tobytes(), pcfg, 4, 8, len(g["train"]))
    assert np.array_equal(st["cursors"], r["cursors"])
    assert np.array_equal(st["hidden"], r["hidden"])
    for a, b in zip(st["params"], r["params"]):
        assert np.array_equal(a, b)
    for a, b in zip(st["opt"], r["opt"]):
        assert np.array_equal(a, b)
    assert st["epoch"] == r["epoch"] and st["eta"] == r["eta"]
    assert st["best"] == r["best_ppl"] and st["bad"] == r["bad_epochs"]


def test_kat_fixture_generators(orc):
    g = load("kat.npz")
    assert np.array_equal(orc.random_stream(1001, 10000, 200)[:200], g["stream_1001"])
    got = np.concatenate([a.ravel()[:16] for a in orc.init_uniform(7, 5, 11)])
    assert np.array_equal(got, g["init_11"])


def test_rmsprop_kats(orc):
    """test_backprop.cpp:585-639 on the oracle."""
    V, H = 6, 4
    params = orc.init_uniform(V, H, 91)
    state = (np.full((H, H), 2.0, np.float32), np.full(V, 3.0, np.float32),
             np.full(V, 5.0, np.float32))
    zero = dict(g_in_words=np.zeros(0, np.uint32), g_in_rows=np.zeros((0, H), np.float32),
                g_rec=np.zeros((H, H), np.float32), g_out_words=np.zeros(0, np.uint32),
                g_out_rows=np.zeros((0, H), np.float32))
    p2, s2, ok = orc.rmsprop(params, state, zero, 0.9, 1e-6, 0.5, out_dense=False)
    assert ok
    for a, b in zip(p2, params):
        assert np.array_equal(a, b)
    assert np.allclose(s2[0], 1.8, atol=1e-7) and np.allclose(s2[1], 2.7, atol=1e-7)
    assert np.allclose(s2[2], 4.5, atol=1e-7)
    # hand computation: m = 0.5*8 + 0.5*12.5 = 10.25
    z = (np.zeros((4, 2), np.float32), np.zeros((2, 2), np.float32), np.zeros((4, 2), np.float32))
    m_in = np.zeros(4, np.float32)
    m_in[2] = 8.0
    g_rec = np.zeros((2, 2), np.float32)
    g_rec[1, 0] = 2.0
    gr = dict(g_in_words=np.array([2], np.uint32), g_in_rows=np.array([[3.0, 4.0]], np.float32),
              g_rec=g_rec, g_out_words=np.zeros(0, np.uint32),
              g_out_rows=np.zeros((0, 2), np.float32))
    p2, s2, ok = orc.rmsprop(z, (np.zeros((2, 2), np.float32), m_in, np.zeros(4, np.float32)),
                             gr, 0.5, 1e-6, 0.1, out_dense=False)
    d = np.sqrt(10.25 + 1e-6)
    assert s2[1][2] == pytest.approx(10.25, abs=1e-5)
    assert p2[0][2, 0] == pytest.approx(-0.1 * 3.0 / d, abs=1e-6)
    assert p2[0][2, 1] == pytest.approx(-0.1 * 4.0 / d, abs=1e-6)
    assert p2[1][1, 0] == pytest.approx(-0.1 * 2.0 / np.sqrt(0.5 * 4 + 1e-6), abs=1e-6)


def test_param_count_kats():
    """test_compress.cpp:60-73 (paper table rows, V = 64,000)."""
    from paper_1502_00512_b200 import param_count
    want = {128: 16400384, 256: 32833536, 512: 65798144, 1024: 132120576,
            2048: 266338304, 4096: 541065216}
    for h, n in want.items():
        assert param_count(64000, h) == n


def test_window_build_cursor_kats(orc):
    """Cursors floor(i*L/N) (test_trainer.cpp:200-251) and the window arrays
    of trainer.hpp:376-387 (modulo-L reads, bos targets masked)."""
    ids = np.arange(100, dtype=np.uint32) % 7
    ids[::6] = 1
    for L, N, want in ((100, 4, [0, 25, 50, 75]), (101, 4, [0, 25, 50, 75])):
        assert [i * L // N for i in range(N)] == want
    assert [i * 259 // 6 for i in range(6)] == [0, 43, 86, 129, 172, 215]
    cur = np.array([0, 25, 50, 97], np.int64)
    x, y, w = orc.window_build(ids, cur, 2, 2, 5)
    for t in range(5):
        for b in range(2):
            pos = cur[2 + b] + t
            assert x[t, b] == ids[pos % 100] and y[t, b] == ids[(pos + 1) % 100]
            assert w[t, b] == (0 if y[t, b] == 1 else 1)


# --------------------------------------- against the reference itself
@pytest.mark.parametrize("seed", range(6))
def test_bptt_random_configs_vs_reference(orc, ref, seed):
    rng = np.random.default_rng(1000 + seed)
    V = int(rng.integers(5, 400))
    H = int(rng.integers(2, 70))
    T = int(rng.integers(1, 9))
    B = int(rng.integers(1, 9))
    act = int(rng.integers(0, 2))
    clip = float([3.4e38, 1.0, 0.01][seed % 3])
    params = ref.init_uniform(V, H, seed)
    x = rng.integers(0, V, (T, B)).astype(np.uint32)
    y = rng.integers(2, V, (T, B)).astype(np.uint32) if V > 2 else x
    w = (rng.random((T, B)) > 0.2).astype(np.uint8)
    h0 = rng.uniform(-0.5, 0.5, (B, H)).astype(np.float32)
    a = orc.bptt(params, act, x, y, w, h0, 1.0 / (T * B), clip)
    b = ref.bptt(params, act, x, y, w, h0, 1.0 / (T * B), clip)
    assert a["loss"] == b["loss"]
    for k in ("h_final", "g_in_words", "g_in_rows", "g_rec", "g_out"):
        assert np.array_equal(a[k], b[k]), k
    st = (rng.uniform(0, 1e-3, (H, H)).astype(np.float32), rng.uniform(0, 1e-3, V).astype(np.float32),
          rng.uniform(0, 1e-3, V).astype(np.float32))
    pa, sa, oka = orc.rmsprop(params, st, a, 0.9995, 1e-6, 0.1)
    pb, sb, okb = ref.rmsprop(params, st, b, 0.9995, 1e-6, 0.1)
    assert oka == okb
    for u, v in zip(pa + sa, pb + sb):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("H,noffset,B,T,L,act", [(8, 2, 2, 5, 400, 0), (6, 3, 1, 4, 257, 1)])
def test_trainer_vs_reference(orc, ref, H, noffset, B, T, L, act):
    from paper_1502_00512_b200 import TrainConfig, formats
    V = 25
    tr, va = ref.random_stream_pair(5 + H, V, L + 16, 100)
    tr = tr[:L]
    params = ref.init_uniform(V, H, 3)
    kw = dict(nstate=H, noffset=noffset, minibatch=B, unroll=T, eta=0.05, max_epochs=4, mode=1,
              act=act)
    blob, logs, ini = ref.train(oracle.TrainConfig(**kw), params, tr, va)
    r = orc.train(oracle.TrainConfig(**kw), params, tr, va)
    assert ini == r["initial_ppl"]
    assert np.array_equal(r["logs"][:, [0, 1, 2, 3, 6]], logs[:, [0, 1, 2, 3, 6]])
    st = formats.read_trainer(blob, TrainConfig(**kw), noffset * B, H, L)
    assert np.array_equal(st["cursors"], r["cursors"])
    for u, v in zip(st["params"] + st["opt"], r["params"] + r["opt"]):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "nce_*.npz"))))
def test_nce_golden_bitexact(orc, path):
    """NCE window (backprop.hpp:126-156): noise model, alias draws from the
    fixture's mt19937_64 state, loss, sparse W_out / W_in rows, W_rec and the
    sparse-W_out rmsprop step all equal the reference's fixture."""
    g = np.load(path)
    params = (g["w_in"], g["w_rec"], g["w_out"])
    noise = orc.noise_build(g["counts"], int(g["k"]), float(g["floor"]))
    st = g["rng0"].copy()
    T, B = g["x"].shape
    r = orc.bptt_nce(params, 0, g["x"], g["y"], g["w"], g["h0"], 1.0 / (T * B), 1.0, noise, st)
    assert np.array_equal(st, g["rng1"])
    assert r["loss"] == float(g["loss"]) and r["positions"] == int(g["positions"])
    for key in ("h_final", "g_in_words", "g_in_rows", "g_rec", "g_out_words", "g_out_rows"):
        assert np.array_equal(r[key], g[key]), key
    state = (g["m_rec"], g["m_in"], g["m_out"])
    p2, s2, ok = orc.rmsprop(params, state, r, 0.9995, 1e-6, 0.05, out_dense=False)
    assert ok == bool(g["applied"])
    for a, key in zip(p2 + s2, ("u_w_in", "u_w_rec", "u_w_out", "u_m_rec", "u_m_in", "u_m_out")):
        assert np.array_equal(a, g[key]), key


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_nce_random_configs_vs_reference(orc, ref, seed):
    rng = np.random.default_rng(seed)
    V, H = int(rng.integers(20, 500)), int(rng.integers(3, 40))
    T, B, k = int(rng.integers(1, 7)), int(rng.integers(1, 6)), int(rng.integers(1, 20))
    act = int(rng.integers(0, 2))
    floor = [1e-8, 1e-3][seed % 2]
    counts = rng.integers(0, 30, V).astype(np.float64)
    counts[1] = 0
    params = orc.init_uniform(V, H, seed)
    x = rng.integers(0, V, (T, B)).astype(np.uint32)
    y = rng.integers(2, V, (T, B)).astype(np.uint32)
    w = (rng.random((T, B)) > 0.2).astype(np.uint8)
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    noise = orc.noise_build(counts, k, floor)
    s1, s2 = orc.mt_state(seed), ref.mt_state(seed)
    assert np.array_equal(s1, s2)
    a = orc.bptt_nce(params, act, x, y, w, h0, 0.1, 0.5, noise, s1)
    b = ref.bptt_nce(params, act, x, y, w, h0, 0.1, 0.5, counts, k, floor, s2)
    assert np.array_equal(s1, s2)
    assert a["loss"] == b["loss"] and a["positions"] == b["positions"]
    for key in ("h_final", "g_in_dense", "g_rec", "g_out_words", "g_out_rows"):
        assert np.array_equal(a[key], b[key]), key


@pytest.mark.parametrize("k,floor,act,eta", [(7, 1e-3, 0, 0.05), (3, 1e-3, 1, 0.005)])
def test_trainer_nce_vs_reference(orc, ref, k, floor, act, eta):
    """Trainer<StandardTraits> in its default NCE mode (trainer.hpp:53,
    207-209, 363-365): the oracle's epochs, final parameters, accumulators,
    cursors and the rng state in the RTRN bytes equal the reference's."""
    from paper_1502_00512_b200 import TrainConfig, formats
    V, H, L = 40, 8, 600
    tr, va = ref.random_stream_pair(77, V, L + 16, 150)
    tr = tr[:L]
    params = ref.init_uniform(V, H, 3)
    kw = dict(nstate=H, noffset=2, minibatch=2, unroll=5, eta=eta, max_epochs=3, mode=0,
              nce_k=k, noise_floor=floor, act=act, divergence_factor=1e9)
    blob, logs, ini = ref.train(oracle.TrainConfig(**kw), params, tr, va)
    r = orc.train(oracle.TrainConfig(**kw), params, tr, va)
    assert ini == r["initial_ppl"]
    assert np.array_equal(r["logs"][:, [0, 1, 2, 3, 6]], logs[:, [0, 1, 2, 3, 6]])
    st = formats.read_trainer(blob, TrainConfig(**kw), 2 * 2, H, L)
    assert np.array_equal(st["cursors"], r["cursors"])
    for u, v in zip(st["params"] + st["opt"], r["params"] + r["opt"]):
        assert np.array_equal(u, v)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "bn_[0-9]*.npz"))))
def test_bottleneck_golden_bitexact(orc, path):
    """Bottleneck model (compress.hpp:38-415): window, bottleneck_update and
    sharded_perplexity of the C restatement equal the reference fixture."""
    g = np.load(path)
    params = (g["e"], g["u"], g["w_rec"], g["d"])
    T, B = g["x"].shape
    r = orc.bn_bptt(params, int(g["act"]), g["x"], g["y"], g["w"], g["h0"], 1.0 / (T * B),
                    float(g["clip"]))
    assert r["loss"] == float(g["loss"]) and r["positions"] == int(g["positions"])
    for key in ("h_final", "g_e", "g_u", "g_rec", "g_d"):
        assert np.array_equal(r[key], g[key]), key
    state = (g["m_e"], g["m_u"], g["m_rec"], g["m_d"])
    p2, s2, ok = orc.bn_update(params, state, r, 0.9995, 1e-6, 0.05)
    assert ok == bool(g["applied"])
    for a, key in zip(p2 + s2, ("u_e", "u_u", "u_w_rec", "u_d", "u_m_e", "u_m_u", "u_m_rec",
                                "u_m_d")):
        assert np.array_equal(a, g[key]), key
    sp = orc.bn_sharded_ppl(params, int(g["act"]), g["ids"], 8)
    assert [sp["total_logprob"], sp["predicted"], sp["perplexity"]] == list(g["sharded"])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_bottleneck_random_configs_vs_reference(orc, ref, seed):
    rng = np.random.default_rng(100 + seed)
    V, H = int(rng.integers(20, 300)), int(rng.integers(4, 40))
    P = int(rng.integers(1, H + 1))
    T, B, act = int(rng.integers(1, 7)), int(rng.integers(1, 6)), int(rng.integers(0, 2))
    pa, pb = orc.bn_init_uniform(V, H, P, seed), ref.bn_init_uniform(V, H, P, seed)
    assert all(np.array_equal(a, b) for a, b in zip(pa, pb))
    x = rng.integers(0, V, (T, B)).astype(np.uint32)
    y = rng.integers(0, V, (T, B)).astype(np.uint32)
    w = (rng.random((T, B)) > 0.2).astype(np.uint8)
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    a = orc.bn_bptt(pa, act, x, y, w, h0, 0.1, 0.5)
    b = ref.bn_bptt(pa, act, x, y, w, h0, 0.1, 0.5)
    assert a["loss"] == b["loss"] and a["positions"] == b["positions"]
    for key in ("h_final", "g_e", "g_u", "g_rec", "g_d"):
        assert np.array_equal(a[key], b[key]), key
    state = tuple(rng.uniform(0, 0.01, s).astype(np.float32) for s in (V, (P, H), (H, H), (H, P)))
    ua, ub = orc.bn_update(pa, state, a, 0.9995, 1e-6, 0.05), ref.bn_update(pa, state, a, 0.9995,
                                                                            1e-6, 0.05)
    assert all(np.array_equal(p, q) for p, q in zip(ua[0] + ua[1], ub[0] + ub[1]))
    # a non-finite gradient rejects the whole update (compress.hpp:300)
    bad = dict(a)
    bad["g_d"] = a["g_d"].copy()
    bad["g_d"].flat[0] = np.nan
    assert not orc.bn_update(pa, state, bad, 0.9995, 1e-6, 0.05)[2]
    ids = orc.random_stream(seed, V, 300)
    assert orc.bn_sharded_ppl(pa, act, ids, 4) == ref.bn_sharded_ppl(pa, act, ids, 4)


@pytest.mark.parametrize("name", ["cycle", "random"])
def test_bottleneck_trainer_golden_bitexact(orc, name):
    """Trainer<BottleneckTraits> restated (oracle bn_train) equals the
    reference's epochs; the package's RTRN writer over the oracle's final
    state reproduces the reference's checkpoint bytes (RNBL + RBOP)."""
    import ast
    from paper_1502_00512_b200 import formats, make_vocab
    g = load(f"bn_train_{name}.npz")
    kw = ast.literal_eval(str(g["cfg"][0]))
    cfg = oracle.TrainConfig(**kw)
    params = (g["e"], g["u"], g["w_rec"], g["d"])
    r = orc.bn_train(cfg, params, g["train"], g["valid"])
    assert r["initial_ppl"] == float(g["initial"])
    cols = [0, 1, 2, 3, 6]
    assert np.array_equal(r["logs"][:, cols], g["logs"][:, cols])
    # the trainer's state after the last epoch (trainer.hpp:262-268): the
    # logged eta is the one the epoch ran with; a non-improving epoch halves it
    logs = r["logs"]
    best_run, bad = float(g["initial"]), 0
    for ppl in logs[:, 2]:
        if ppl < best_run:
            best_run, bad = ppl, 0
        else:
            bad += 1
    eta = float(logs[-1, 3]) * (0.5 if bad else 1.0)
    blob = formats.write_trainer(cfg, len(logs), eta, best_run, bad, float(g["initial"]),
                                 formats.mt19937_64_text(cfg.seed), r["cursors"], r["hidden"],
                                 r["params"], make_vocab(int(g["e"].shape[0])), r["opt"],
                                 model="bottleneck")
    assert blob == g["rtrn"].tobytes()


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "bn_nce_*.npz"))))
def test_bottleneck_nce_golden_bitexact(orc, path):
    """Bottleneck model, NCE mode: draws, loss, the sparse embedding rows in
    slot order and the sparse-embedding bottleneck_update equal the
    reference fixture."""
    g = np.load(path)
    params = (g["e"], g["u"], g["w_rec"], g["d"])
    T, B = g["x"].shape
    noise = orc.noise_build(g["counts"], int(g["k"]), float(g["floor"]))
    st = g["rng0"].copy()
    r = orc.bn_bptt_nce(params, int(g["act"]), g["x"], g["y"], g["w"], g["h0"], 1.0 / (T * B),
                        1.0, noise, st)
    assert np.array_equal(st, g["rng1"])
    assert r["loss"] == float(g["loss"]) and r["positions"] == int(g["positions"])
    for key in ("h_final", "g_e_words", "g_e_rows", "g_u", "g_rec", "g_d"):
        assert np.array_equal(r[key], g[key]), key
    state = (g["m_e"], g["m_u"], g["m_rec"], g["m_d"])
    p2, s2, ok = orc.bn_update_sparse(params, state, r, 0.9995, 1e-6, 0.05)
    assert ok == bool(g["applied"])
    for a, key in zip(p2 + s2, ("u_e", "u_u", "u_w_rec", "u_d", "u_m_e", "u_m_u", "u_m_rec",
                                "u_m_d")):
        assert np.array_equal(a, g[key]), key


def test_bottleneck_trainer_nce_golden(orc):
    """Trainer<BottleneckTraits> in its default NCE mode: epochs and the
    RTRN checkpoint (generator state included) equal the reference's."""
    import ast
    from paper_1502_00512_b200 import formats, make_vocab
    g = load("bn_train_nce.npz")
    kw = ast.literal_eval(str(g["cfg"][0]))
    cfg = oracle.TrainConfig(**kw)
    params = (g["e"], g["u"], g["w_rec"], g["d"])
    r = orc.bn_train(cfg, params, g["train"], g["valid"])
    cols = [0, 1, 2, 3, 6]
    assert r["initial_ppl"] == float(g["initial"])
    assert np.array_equal(r["logs"][:, cols], g["logs"][:, cols])
    logs = r["logs"]
    best, bad = float(g["initial"]), 0
    for ppl in logs[:, 2]:
        if ppl < best:
            best, bad = ppl, 0
        else:
            bad += 1
    eta = float(logs[-1, 3]) * (0.5 if bad else 1.0)
    rng_text = " ".join(str(int(v)) for v in r["rng"])
    blob = formats.write_trainer(cfg, len(logs), eta, best, bad, float(g["initial"]), rng_text,
                                 r["cursors"], r["hidden"], r["params"],
                                 make_vocab(int(g["e"].shape[0])), r["opt"], model="bottleneck")
    assert blob == g["rtrn"].tobytes()


def test_ln_z_samples_golden_and_drift_stats(orc):
    """ln_z_samples (eval.hpp:805-857) restated bit-exact; the package's
    host drift_stats (eval.hpp:859-880) equals the reference's."""
    import paper_1502_00512_b200 as dl
    g = load("ln_z.npz")
    params = (g["w_in"], g["w_rec"], g["w_out"])
    z = orc.ln_z_samples(params, int(g["act"]), g["ids"], int(g["count"]))
    assert np.array_equal(z, g["ln_z"])
    s = dl.drift_stats(z)
    assert [s.mean, s.median, s.q25, s.q75, s.iqr, s.contexts] == list(g["stats"])
    with pytest.raises(ValueError):
        dl.drift_stats(z[:99])
