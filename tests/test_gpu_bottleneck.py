"""GPU parity of the bottleneck / tied-embedding model (compress.hpp:38-415)
against the C oracle and the reference's fixtures, through the C ABI
(dl_bn_*): one softmax window (loss, h_final, the four clipped gradients),
bottleneck_update, sharded_perplexity, and a short training run.

fp32 mode: the GEMMs accumulate in fp32 where the reference uses double,
so agreement is to summation order (1e-4 relative, as the standard model).
bf16 mode: tensor-core operands; compared by loss / perplexity (1%) and
gradient direction (cosine)."""
import glob
import os

import numpy as np
import pytest

from test_gpu_window import close, rand_window

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

CASES = [
    # V, H, P, T, B, act, mask, clip
    (7, 5, 3, 4, 2, 0, 0.15, 3.4e38),
    (60, 16, 8, 5, 4, 1, 0.2, 0.05),
    (333, 64, 16, 8, 8, 0, 0.1, 1.0),
    (2000, 128, 64, 8, 16, 0, 0.1, 1.0),
    (10000, 128, 32, 8, 8, 1, 0.1, 1.0),
]


def bn_model(dl_bn, params, act, precision):
    V, P = params[0].shape
    H = params[2].shape[0]
    m = dl_bn.GpuBottleneck(V, H, P, act, precision)
    m.set_params(*params)
    return m


@pytest.mark.parametrize("V,H,P,T,B,act,mask,clip", CASES)
def test_bn_window_fp32_matches_oracle(orc, V, H, P, T, B, act, mask, clip):
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    rng = np.random.default_rng(V + P)
    params = orc.bn_init_uniform(V, H, P, 3)
    x, y, w = rand_window(rng, T, B, V, mask)
    h0 = rng.uniform(-0.5, 0.5, (B, H)).astype(np.float32)
    scale = 1.0 / (T * B)
    want = orc.bn_bptt(params, act, x, y, w, h0, scale, clip)
    m = bn_model(bn, params, act, "fp32")
    res, hf = bn.bn_bptt_run(m, dl.WindowBatch(x, y, w), h0, scale, clip)
    assert res.positions == want["positions"]
    assert res.loss == pytest.approx(want["loss"], rel=1e-6)
    ok, err = close(hf, want["h_final"])
    assert ok, err
    for got, key in zip(m.grads(), ("g_e", "g_u", "g_rec", "g_d")):
        ok, err = close(got, want[key])
        assert ok, (key, err)
    # bottleneck_update given the same gradients
    state = (np.zeros(V, np.float32), np.zeros((P, H), np.float32),
             np.zeros((H, H), np.float32), np.zeros((H, P), np.float32))
    p2, s2, ok = orc.bn_update(params, state, want, 0.9995, 1e-6, 0.05)
    assert bn.bottleneck_update(m, 0.05) == ok
    for a, b in zip(m.params() + m.opt(), p2 + s2):
        ok_, err = close(a, b, rel=1e-4, floor_frac=1e-5)
        assert ok_, err


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "bn_[0-9]*.npz"))))
def test_bn_window_matches_reference_fixture(path):
    """Against the reference's own BottleneckAdapter window and update."""
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    g = np.load(path)
    params = (g["e"], g["u"], g["w_rec"], g["d"])
    T, B = g["x"].shape
    m = bn_model(bn, params, int(g["act"]), "fp32")
    m.set_opt(g["m_e"], g["m_u"], g["m_rec"], g["m_d"])
    res, hf = bn.bn_bptt_run(m, dl.WindowBatch(g["x"], g["y"], g["w"]), g["h0"], 1.0 / (T * B),
                             float(g["clip"]))
    assert res.positions == int(g["positions"])
    assert res.loss == pytest.approx(float(g["loss"]), rel=1e-6)
    assert close(hf, g["h_final"])[0]
    for got, key in zip(m.grads(), ("g_e", "g_u", "g_rec", "g_d")):
        ok, err = close(got, g[key])
        assert ok, (key, err)
    assert bn.bottleneck_update(m, 0.05) == bool(g["applied"])
    for got, key in zip(m.params() + m.opt(), ("u_e", "u_u", "u_w_rec", "u_d", "u_m_e", "u_m_u",
                                                "u_m_rec", "u_m_d")):
        ok, err = close(got, g[key], rel=1e-4, floor_frac=1e-5)
        assert ok, (key, err)
    r = bn.bn_sharded_perplexity(m, g["ids"], 8)  # (updated params: only check it runs)
    assert r.predicted == int(g["sharded"][1])


@pytest.mark.parametrize("V,H,P,act,shards", [(60, 16, 8, 0, 8), (500, 64, 32, 1, 16),
                                              (4096, 256, 128, 0, 64)])
def test_bn_sharded_perplexity_matches_oracle(orc, V, H, P, act, shards):
    from paper_1502_00512_b200 import bottleneck as bn
    params = orc.bn_init_uniform(V, H, P, 5)
    ids = orc.random_stream(77, V, 3000)
    want = orc.bn_sharded_ppl(params, act, ids, shards)
    m = bn_model(bn, params, act, "fp32")
    r = bn.bn_sharded_perplexity(m, ids, shards)
    assert r.predicted == want["predicted"]
    assert r.total_logprob == pytest.approx(want["total_logprob"], rel=1e-5)
    assert r.perplexity == pytest.approx(want["perplexity"], rel=1e-4)


def test_bn_nonfinite_gradient_skips_update(orc):
    """bottleneck_update returns false on a non-finite gradient and leaves
    parameters and accumulators untouched (compress.hpp:300)."""
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    V, H, P, T, B = 40, 8, 4, 3, 2
    params = list(orc.bn_init_uniform(V, H, P, 1))
    params[3] = params[3].copy()
    params[3][0, 0] = np.inf  # D: an infinite score -> NaN gradients
    rng = np.random.default_rng(0)
    x, y, w = rand_window(rng, T, B, V, 0.0)
    m = bn_model(bn, tuple(params), 0, "fp32")
    h0 = np.zeros((B, H), np.float32)
    # an infinite clip bound keeps the non-finite values (a NaN clipped at a
    # finite bound becomes -clip, rnn.hpp:131-134)
    want = orc.bn_bptt(tuple(params), 0, x, y, w, h0, 0.1, np.inf)
    st0 = (np.zeros(V, np.float32), np.zeros((P, H), np.float32), np.zeros((H, H), np.float32),
           np.zeros((H, P), np.float32))
    assert not orc.bn_update(tuple(params), st0, want, 0.9995, 1e-6, 0.05)[2]
    bn.bn_bptt_run(m, dl.WindowBatch(x, y, w), h0, 0.1, np.inf)
    before = m.params() + m.opt()
    assert not bn.bottleneck_update(m, 0.05)
    for a, b in zip(m.params() + m.opt(), before):
        assert np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("V,H,P,T,B,act", [(4096, 256, 64, 8, 32, 0), (8192, 512, 128, 16, 64, 0),
                                            (4096, 256, 128, 8, 16, 1)])
def test_bn_window_bf16_close_to_oracle(orc, V, H, P, T, B, act):
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    rng = np.random.default_rng(V)
    params = orc.bn_init_uniform(V, H, P, 4)
    x, y, w = rand_window(rng, T, B, V, 0.1)
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    want = orc.bn_bptt(params, act, x, y, w, h0, 1.0 / (T * B), 1.0)
    m = bn_model(bn, params, act, "bf16")
    res, hf = bn.bn_bptt_run(m, dl.WindowBatch(x, y, w), h0, 1.0 / (T * B), 1.0)
    assert res.loss == pytest.approx(want["loss"], rel=1e-2)
    assert np.max(np.abs(hf - want["h_final"])) < 2e-2
    for got, key in zip(m.grads(), ("g_e", "g_u", "g_rec", "g_d")):
        ref = want[key]
        cos = float(np.dot(got.ravel(), ref.ravel()) /
                    (np.linalg.norm(got) * np.linalg.norm(ref) + 1e-30))
        assert cos > 0.99, (key, cos)
    assert bn.bottleneck_update(m, 0.01)
    ids = orc.random_stream(9, V, 20000)
    r = bn.bn_sharded_perplexity(m, ids, 64)
    p2 = m.params()
    want_p = orc.bn_sharded_ppl(p2, act, ids, 64)
    assert r.perplexity == pytest.approx(want_p["perplexity"], rel=1e-2)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_bn_training_windows_follow_oracle(orc, precision):
    """Several consecutive windows of bptt_run + bottleneck_update (the
    Trainer's step) on the device follow the oracle's trajectory."""
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    V, H, P, T, B = 512, 64, 32, 8, 16
    rng = np.random.default_rng(3)
    params = orc.bn_init_uniform(V, H, P, 9)
    m = bn_model(bn, params, 0, precision)
    state = (np.zeros(V, np.float32), np.zeros((P, H), np.float32),
             np.zeros((H, H), np.float32), np.zeros((H, P), np.float32))
    cur = params
    h = np.full((B, H), 0.5, np.float32)
    hw = h.copy()
    # (eta 0.05 diverges on this random-data model within a few windows --
    # the loss grows 100x -- and the chaotic trajectory amplifies rounding)
    eta = 0.005
    for i in range(6):
        x, y, w = rand_window(rng, T, B, V, 0.1)
        want = orc.bn_bptt(cur, 0, x, y, w, hw, 1.0 / (T * B), 1.0)
        cur, state, ok = orc.bn_update(cur, state, want, 0.9995, 1e-6, eta)
        hw = want["h_final"]
        res, h, applied = bn.bn_train_window(m, dl.WindowBatch(x, y, w), h, 1.0 / (T * B), 1.0,
                                             eta)
        assert applied and ok
        assert res.loss == pytest.approx(want["loss"], rel=1e-4 if precision == "fp32" else 2e-2)
    if precision == "fp32":
        for a, b in zip(m.params(), cur):
            assert np.mean(np.abs(a - b)) < 1e-4 * np.mean(np.abs(b))


@pytest.mark.parametrize("name", ["random", "cycle"])
def test_bn_trainer_matches_reference_fixture(name):
    """BottleneckTrainer (device windows, host schedule) against the
    reference's Trainer<BottleneckTraits> epochs (tests/golden/bn_train_*),
    then a checkpoint round trip that resumes bit-for-bit."""
    import ast
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    g = np.load(os.path.join(GOLD, f"bn_train_{name}.npz"))
    kw = ast.literal_eval(str(g["cfg"][0]))
    cfg = dl.TrainConfig(**kw)
    params = (g["e"], g["u"], g["w_rec"], g["d"])
    V = params[0].shape[0]
    t = bn.BottleneckTrainer(cfg, params, dl.make_vocab(V), g["train"], g["valid"])
    t.train()
    assert t.initial_ppl == pytest.approx(float(g["initial"]), rel=1e-5)
    want = g["logs"]
    if name == "random":
        assert len(t.logs) == len(want)
        for a, b in zip(t.logs, want):
            assert a.train_loss == pytest.approx(b[1], rel=1e-4)
            assert a.valid_ppl == pytest.approx(b[2], rel=1e-4)
            assert a.eta == b[3]
    else:
        # the reference's own test (test_compress.cpp:427-446): 30 epochs on
        # a deterministic cycle must drive validation perplexity below 1.3.
        # (At eta 0.02 the first rmsprop steps move weights by ~eta each, so
        # the trajectory is chaotic: summation-order differences already show
        # in the first epoch, and the -ffp-contract=off reference build of
        # the fixture stalls at 1.48 -- only the test's criterion is shared.)
        assert t.best_ppl < 1.3
    blob = t.save_checkpoint()
    t2 = bn.BottleneckTrainer(cfg, params, dl.make_vocab(V), g["train"], g["valid"])
    t2.load_checkpoint(blob)
    assert t2.save_checkpoint() == blob
    assert len(blob) == len(g["rtrn"])


# ----------------------------------------------------------------- NCE mode
def bn_nce_model(bn, params, counts, k, floor, precision, act=0, state=None):
    m = bn_model(bn, params, act, precision)
    m.set_loss_mode(0)
    m.set_noise(counts, k, floor)
    m.set_rng_state(state)
    return m


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "bn_nce_*.npz"))))
def test_bn_nce_window_matches_reference_fixture(path):
    """NCE window over the bottleneck adapter against the reference's own:
    the generator state after the draws, loss, the sparse embedding
    gradient (dense view) and the sparse-embedding update."""
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    g = np.load(path)
    params = (g["e"], g["u"], g["w_rec"], g["d"])
    V, P = params[0].shape
    T, B = g["x"].shape
    m = bn_nce_model(bn, params, g["counts"], int(g["k"]), float(g["floor"]), "fp32",
                     int(g["act"]), g["rng0"])
    m.set_opt(g["m_e"], g["m_u"], g["m_rec"], g["m_d"])
    res, hf = bn.bn_bptt_run(m, dl.WindowBatch(g["x"], g["y"], g["w"]), g["h0"], 1.0 / (T * B),
                             1.0)
    assert np.array_equal(m.rng_state(), g["rng1"])
    assert res.positions == int(g["positions"])
    assert res.loss == pytest.approx(float(g["loss"]), rel=1e-6)
    assert close(hf, g["h_final"])[0]
    g_e = np.zeros((V, P), np.float32)
    g_e[g["g_e_words"]] = g["g_e_rows"]
    for got, want in zip(m.grads(), (g_e, g["g_u"], g["g_rec"], g["g_d"])):
        ok, err = close(got, want)
        assert ok, err
    assert bn.bottleneck_update(m, 0.05) == bool(g["applied"])
    for got, key in zip(m.params() + m.opt(), ("u_e", "u_u", "u_w_rec", "u_d", "u_m_e", "u_m_u",
                                                "u_m_rec", "u_m_d")):
        ok, err = close(got, g[key], rel=1e-4, floor_frac=1e-5)
        assert ok, (key, err)


@pytest.mark.parametrize("V,H,P,T,B,k,act", [(504, 64, 32, 6, 8, 16, 1), (4096, 256, 64, 8, 32, 32, 0)])
def test_bn_nce_window_matches_oracle(orc, V, H, P, T, B, k, act):
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    rng = np.random.default_rng(V + k)
    params = orc.bn_init_uniform(V, H, P, 2)
    counts = rng.integers(0, 50, V).astype(np.float64)
    x, y, w = rand_window(rng, T, B, V, 0.1)
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    noise = orc.noise_build(counts, k, 1e-8)
    st = orc.mt_state(11)
    want = orc.bn_bptt_nce(params, act, x, y, w, h0, 1.0 / (T * B), 1.0, noise, st)
    for precision in ("fp32", "bf16"):
        m = bn_nce_model(bn, params, counts, k, 1e-8, precision, act, orc.mt_state(11))
        res, hf = bn.bn_bptt_run(m, dl.WindowBatch(x, y, w), h0, 1.0 / (T * B), 1.0)
        assert np.array_equal(m.rng_state(), st)
        if precision == "fp32":
            assert res.loss == pytest.approx(want["loss"], rel=1e-6)
            for got, key in zip(m.grads(), ("g_e", "g_u", "g_rec", "g_d")):
                ok, err = close(got, want[key])
                assert ok, (key, err)
        else:
            assert res.loss == pytest.approx(want["loss"], rel=1e-2)
            ge = m.grads()[0]
            cos = float(np.dot(ge.ravel(), want["g_e"].ravel()) /
                        (np.linalg.norm(ge) * np.linalg.norm(want["g_e"]) + 1e-30))
            assert cos > 0.99


def test_bn_trainer_nce_matches_reference_fixture():
    """BottleneckTrainer in NCE mode (the reference Trainer default) against
    the reference's epochs; the generator advances exactly as the
    reference's and the checkpoint resumes bit-for-bit."""
    import ast
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    g = np.load(os.path.join(GOLD, "bn_train_nce.npz"))
    kw = ast.literal_eval(str(g["cfg"][0]))
    cfg = dl.TrainConfig(**kw)
    params = (g["e"], g["u"], g["w_rec"], g["d"])
    V = params[0].shape[0]
    t = bn.BottleneckTrainer(cfg, params, dl.make_vocab(V), g["train"], g["valid"])
    t.train()
    want = g["logs"]
    assert t.initial_ppl == pytest.approx(float(g["initial"]), rel=1e-5)
    assert len(t.logs) == len(want)
    for a, b in zip(t.logs, want):
        assert a.train_loss == pytest.approx(b[1], rel=1e-4)
        assert a.valid_ppl == pytest.approx(b[2], rel=1e-4)
    blob = t.save_checkpoint()
    assert len(blob) == len(g["rtrn"])
    # same draws made (generator state), same schedule (cursors)
    from paper_1502_00512_b200 import formats
    L = len(g["train"])
    mine = formats.read_trainer(blob, cfg, len(t.cursors), t.model.H, L, model="bottleneck")
    ref = formats.read_trainer(g["rtrn"].tobytes(), cfg, len(t.cursors), t.model.H, L,
                               model="bottleneck")
    assert mine["rng_text"] == ref["rng_text"]
    assert np.array_equal(mine["cursors"], ref["cursors"])
    assert (mine["epoch"], mine["eta"], mine["bad"]) == (ref["epoch"], ref["eta"], ref["bad"])
    t2 = bn.BottleneckTrainer(cfg, params, dl.make_vocab(V), g["train"], g["valid"])
    t2.load_checkpoint(blob)
    assert t2.save_checkpoint() == blob


@pytest.mark.parametrize("bits", [3, 8, 13])
def test_rnqz_device_dequantization_bitexact(bits, orc):
    """RNQZ -> device dequantisation (dl_bn_set_params_quantized) gives the
    reference's dequantized parameters bit for bit; the scorer then runs on
    them (sharded perplexity vs the oracle)."""
    from paper_1502_00512_b200 import bottleneck as bn, formats
    g = np.load(os.path.join(GOLD, "rnqz.npz"))
    q = formats.read_quantized(g[f"rnqz_{bits}"].tobytes())
    m = bn.GpuBottleneck(q.v, q.h, q.p, q.act, "fp32")
    m.set_params_quantized(q)
    got = m.params()
    for a, k in zip(got, ("e", "u", "w_rec", "d")):
        assert np.array_equal(a, g[f"dq_{bits}_{k}"]), k
    ids = orc.random_stream(5, q.v, 2000)
    want = orc.bn_sharded_ppl(got, q.act, ids, 8)
    r = bn.bn_sharded_perplexity(m, ids, 8)
    assert r.perplexity == pytest.approx(want["perplexity"], rel=1e-4)


@pytest.mark.parametrize("precision,mode", [("fp32", 1), ("bf16", 1), ("fp32", 0), ("bf16", 0)])
def test_bn_device_epoch_loop_matches_host_schedule(orc, precision, mode):
    """dl_bn_trainer_run (the epoch's windows built, trained and carried on
    the device; softmax windows from one CUDA graph) against the host-side
    schedule driving dl_bn_train_window per window: the same windows in the
    same order, so logs, parameters, optimiser state, cursors, hidden carry
    and the generator are bit-identical; then a checkpoint written by one
    resumes in the other."""
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    V, H, P = 512, 64, 32
    tr, va = orc.random_stream_pair(17, V, 6000, 800)
    params = orc.bn_init_uniform(V, H, P, 4)
    # (the comparison is between the two schedules, not about convergence:
    # no divergence stop)
    cfg = dl.TrainConfig(nstate=H, nproj=P, noffset=3, minibatch=8, unroll=6,
                         eta=0.02 if mode == 1 else 0.004, mode=mode, nce_k=8, max_epochs=2,
                         seed=3, divergence_factor=1e30)
    runs = []
    for device_loop in (True, False):
        t = bn.BottleneckTrainer(cfg, params, dl.make_vocab(V), tr, va, precision,
                                 device_loop=device_loop)
        t.train()
        runs.append(t)
    a, b = runs
    assert [(l.train_loss, l.valid_ppl, l.eta) for l in a.logs] == \
        [(l.train_loss, l.valid_ppl, l.eta) for l in b.logs]
    for x, y in zip(a.model.params() + a.model.opt(), b.model.params() + b.model.opt()):
        assert np.array_equal(x, y)
    assert np.array_equal(a.cursors, b.cursors)
    assert np.array_equal(a.hidden, b.hidden)
    assert np.array_equal(a.model.rng_state(), b.model.rng_state())
    blob = a.save_checkpoint()
    assert blob == b.save_checkpoint()
    c = bn.BottleneckTrainer(cfg, params, dl.make_vocab(V), tr, va, precision,
                             device_loop=False)
    c.load_checkpoint(blob)
    assert c.save_checkpoint() == blob
    # one more epoch each from the same state: still identical
    a.eta = c.eta = 0.01
    la, lc = a.run_epoch(), c.run_epoch()
    assert la == lc
    for x, y in zip(a.model.params(), c.model.params()):
        assert np.array_equal(x, y)


def test_bn_device_epoch_loop_errors():
    from paper_1502_00512_b200 import DataError, bottleneck as bn
    m = bn.GpuBottleneck(64, 16, 8, 0, "fp32")
    with pytest.raises(ValueError):
        m.trainer_run(0, 1, 0.1)  # not initialised
    with pytest.raises(ValueError):
        m.trainer_init(np.arange(10, dtype=np.uint32), 4, 4, 2, 1.0)  # L < N
    with pytest.raises(DataError):
        m.trainer_init(np.full(100, 64, np.uint32), 2, 2, 2, 1.0)  # id >= V
    m.trainer_init(np.arange(100, dtype=np.uint32) % 64, 2, 2, 2, 1.0)
    with pytest.raises(DataError):
        m.trainer_set_state(np.full(4, 100, np.int64), np.zeros((4, 16), np.float32))
    m.close()
