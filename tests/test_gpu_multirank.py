"""The multi-rank code paths run on ONE GPU: G contexts in one process form
an in-process rank group (dl_local_group_create / dl_comm_init_local, the
same collective interface the NCCL path implements), one host thread per
rank.  Data parallel: every rank trains its slice of the
global minibatch; gradients are summed before clip + rmsprop, so replicas
must stay bit-identical and equal a single context training the whole
global minibatch (to fp32 summation-order tolerance)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def close(a, b, rel=1e-4):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= rel * np.abs(b) + 1e-4 * np.abs(b).max())


@pytest.mark.parametrize("G,precision", [(2, "fp32"), (4, "fp32"), (2, "bf16")])
def test_dp_window_matches_global_window(orc, G, precision):
    import paper_1502_00512_b200 as dl
    V, H, T, B = 512, 64, 6, 8
    Bg = G * B
    rng = np.random.default_rng(G)
    params = orc.init_uniform(V, H, 21)
    x = rng.integers(0, V, (T, Bg)).astype(np.uint32)
    y = rng.integers(2, V, (T, Bg)).astype(np.uint32)
    w = (rng.random((T, Bg)) > 0.1).astype(np.uint8)
    h0 = rng.uniform(0, 1, (Bg, H)).astype(np.float32)
    scale = 1.0 / (Bg * T)
    single = dl.GpuRnn(V, H, 0, precision)
    single.set_params(*params)
    r1, hf1 = dl.bptt_run(single, dl.WindowBatch(x, y, w), h0, scale, 1.0)
    assert dl.rmsprop_update(single, 0.05)
    want = single.params() + single.opt()

    group = dl.LocalGroup(G)
    ranks = []
    for r in range(G):
        m = dl.GpuRnn(V, H, 0, precision)
        m.comm_init_local(group, r)
        m.set_params(*params)
        ranks.append(m)

    def run(r):
        sl = slice(r * B, (r + 1) * B)
        wb = dl.WindowBatch(np.ascontiguousarray(x[:, sl]), np.ascontiguousarray(y[:, sl]),
                            np.ascontiguousarray(w[:, sl]))
        res, hf = dl.bptt_run(ranks[r], wb, np.ascontiguousarray(h0[sl]), scale, 1.0)
        ok = dl.rmsprop_update(ranks[r], 0.05)
        return res, hf, ok

    with ThreadPoolExecutor(G) as ex:
        outs = list(ex.map(run, range(G)))
    for r, (res, hf, ok) in enumerate(outs):
        assert ok
        assert res.loss == pytest.approx(r1.loss, rel=1e-6)  # global (allreduced) loss
        assert res.positions == r1.positions
        assert np.allclose(hf, hf1[r * B:(r + 1) * B], atol=1e-6 if precision == "fp32" else 2e-2)
    got = [m.params() + m.opt() for m in ranks]
    for r in range(1, G):  # replicas are bit-identical
        for a, b in zip(got[0], got[r]):
            assert np.array_equal(a, b)
    if precision == "fp32":
        for a, b in zip(got[0], want):
            assert close(a, b)
    else:
        # bf16: dW_out is summed over ranks in bf16 before clip + update
        for a, b in zip(got[0][:3], want[:3]):
            d = np.asarray(a, np.float64) - np.asarray(b, np.float64)
            assert np.abs(d).max() <= 2e-2 * max(1.0, np.abs(b).max())


def _vshard_ranks(dl, G, V, H, precision, params):
    group = dl.LocalGroup(G)
    ranks = []
    for r in range(G):
        m = dl.GpuRnn(V, H, 0, precision)
        m.comm_init_local(group, r)
        m.set_vocab_shard(True)
        m.set_params(*params)
        ranks.append(m)
    return ranks


def _assemble(parts, G):
    """Row block r of the vocabulary-sharded arrays comes from rank r."""
    V = parts[0].shape[0]
    out = np.zeros_like(parts[0])
    for r in range(G):
        out[r * V // G:(r + 1) * V // G] = parts[r][r * V // G:(r + 1) * V // G]
    return out


@pytest.mark.parametrize("G,precision", [(2, "fp32"), (4, "fp32"), (2, "bf16"), (4, "bf16")])
def test_vocab_shard_window_matches_full_softmax(orc, G, precision):
    """G ranks each own V/G rows of W_out; loss, h_final,
    gradients and the updated parameters equal one context holding the whole
    output layer (fp32: 1e-5, the two-level log-sum-exp is the only change;
    bf16: the same tensor-core tiles over a narrower N)."""
    import paper_1502_00512_b200 as dl
    V, H, T, B = 1024, 64, 6, 16
    rng = np.random.default_rng(7 + G)
    params = orc.init_uniform(V, H, 31)
    x = rng.integers(0, V, (T, B)).astype(np.uint32)
    y = rng.integers(2, V, (T, B)).astype(np.uint32)
    w = (rng.random((T, B)) > 0.1).astype(np.uint8)
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    scale = 1.0 / (B * T)
    wb = dl.WindowBatch(x, y, w)
    single = dl.GpuRnn(V, H, 0, precision)
    single.set_params(*params)
    r1, hf1 = dl.bptt_run(single, wb, h0, scale, 1.0)
    g1 = single.grads()
    assert dl.rmsprop_update(single, 0.05)
    want = single.params() + single.opt()

    ranks = _vshard_ranks(dl, G, V, H, precision, params)

    def run(r):
        res, hf = dl.bptt_run(ranks[r], wb, h0, scale, 1.0)
        g = ranks[r].grads()
        ok = dl.rmsprop_update(ranks[r], 0.05)
        return res, hf, g, ok

    with ThreadPoolExecutor(G) as ex:
        outs = list(ex.map(run, range(G)))
    tol = 1e-5 if precision == "fp32" else 2e-3
    for res, hf, g, ok in outs:
        assert ok
        assert res.positions == r1.positions
        assert res.loss == pytest.approx(r1.loss, rel=tol)
        assert np.allclose(hf, hf1, atol=1e-6)  # forward recurrence is replicated
        assert res.loss == outs[0][0].loss  # every rank reports the same loss
    # replicated state (W_in, W_rec, their grads) is bit-identical across ranks
    got = [m.params() + m.opt() for m in ranks]
    for r in range(1, G):
        for k in (0, 1, 3, 4):
            assert np.array_equal(got[0][k], got[r][k])
        for k in (0, 1):
            assert np.array_equal(outs[0][2][k], outs[r][2][k])
    g_out = _assemble([o[2][2] for o in outs], G)
    w_out = _assemble([gr[2] for gr in got], G)
    m_out = _assemble([gr[5][:, None] for gr in got], G)[:, 0]
    if precision == "fp32":
        for a, b in zip(outs[0][2][:2] + (g_out,), g1):
            assert close(a, b, 1e-5)
        for a, b in zip(got[0][:2] + (w_out,) + got[0][3:5] + (m_out,), want):
            assert close(a, b, 1e-5)
    else:
        # bf16: dW_out within bf16 rounding of the single-context gradient
        assert np.abs(g_out - g1[2]).max() <= 2e-2 * np.abs(g1[2]).max()
        assert np.abs(w_out - want[2]).max() <= 1e-3


def test_vocab_shard_scoring_and_trainer(orc):
    """Sharded scoring equals full scoring; a vocab-sharded trainer tracks
    the single-context trainer (same streams on every rank)."""
    import paper_1502_00512_b200 as dl
    V, H, G = 96, 32, 2
    tr, va = orc.random_stream_pair(23, V, 3016, 600)
    tr = tr[:3000]
    params = orc.init_uniform(V, H, 5)
    single = dl.GpuRnn(V, H, 0, "fp32")
    single.set_params(*params)
    want = dl.sharded_perplexity(single, va, 4)
    ranks = _vshard_ranks(dl, G, V, H, "fp32", params)
    with ThreadPoolExecutor(G) as ex:
        got = list(ex.map(lambda m: dl.sharded_perplexity(m, va, 4), ranks))
    for p in got:
        assert p.predicted == want.predicted
        assert p.total_logprob == pytest.approx(want.total_logprob, rel=1e-9)

    kw = dict(nstate=H, noffset=2, minibatch=4, unroll=5, eta=0.02, max_epochs=2, mode=1)
    ref = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, "fp32")
    ref.train()
    group = dl.LocalGroup(G)
    trainers = [dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, "fp32",
                           comm=(group, G, r), vocab_shard=True) for r in range(G)]
    with ThreadPoolExecutor(G) as ex:
        list(ex.map(lambda t: t.train(), trainers))
    for t in trainers:
        assert len(t.logs) == len(ref.logs)
        for a, b in zip(t.logs, ref.logs):
            assert a.train_loss == pytest.approx(b.train_loss, rel=1e-4)
            assert a.valid_ppl == pytest.approx(b.valid_ppl, rel=1e-3)
    w_out = _assemble([t.params()[2] for t in trainers], G)
    assert close(w_out, ref.params()[2], 1e-2)


def test_dp_trainer_matches_global_minibatch(orc):
    """Two ranks x minibatch 4 == one trainer with minibatch 8 (same
    schedule: rank r owns streams g*8 + r*4 + b)."""
    import paper_1502_00512_b200 as dl
    V, H, G = 80, 32, 2
    tr, va = orc.random_stream_pair(17, V, 4016, 600)
    tr = tr[:4000]
    params = orc.init_uniform(V, H, 9)
    kw = dict(nstate=H, noffset=3, unroll=5, eta=0.02, max_epochs=2, mode=1)
    single = dl.Trainer(dl.TrainConfig(minibatch=G * 4, **kw), params, dl.make_vocab(V), tr, va,
                        "fp32")
    single.train()
    group = dl.LocalGroup(G)
    trainers = [dl.Trainer(dl.TrainConfig(minibatch=4, **kw), params, dl.make_vocab(V), tr, va,
                           "fp32", comm=(group, G, r)) for r in range(G)]
    with ThreadPoolExecutor(G) as ex:
        list(ex.map(lambda t: t.train(), trainers))
    for t in trainers:
        assert len(t.logs) == len(single.logs)
        for a, b in zip(t.logs, single.logs):
            assert a.train_loss == pytest.approx(b.train_loss, rel=1e-4)
            assert a.valid_ppl == pytest.approx(b.valid_ppl, rel=1e-3)
    # cursors: rank r's group-major slice interleaves into the global layout
    cs, _ = single.model.trainer_state()
    Bg, nof = G * 4, 3
    for r, t in enumerate(trainers):
        c, _ = t.model.trainer_state()
        for g in range(nof):
            assert np.array_equal(c[g * 4:(g + 1) * 4], cs[g * Bg + r * 4:g * Bg + (r + 1) * 4])
    for a, b in zip(trainers[0].params(), trainers[1].params()):
        assert np.array_equal(a, b)
    # a rank holds only its streams' state: no single-rank RTRN blob
    with pytest.raises(NotImplementedError):
        trainers[0].save_checkpoint()


@pytest.mark.parametrize("G", [2, 3])
def test_dp_nce_trainer_matches_global_minibatch(orc, G):
    """NCE (LossMode::kNce, the reference's default) under data-parallel
    ranks: the noise of the global window is drawn in the reference's
    (t, global stream, sample) order from one generator -- identical on every
    rank -- so G ranks x minibatch 4 train exactly like one trainer with
    minibatch 4G (trainer.hpp:53, backprop.hpp:126-156)."""
    import paper_1502_00512_b200 as dl
    V, H = 60, 16
    tr, va = orc.random_stream_pair(23, V, 3016, 400)
    tr = tr[:3000]
    params = orc.init_uniform(V, H, 11)
    kw = dict(nstate=H, noffset=3, unroll=5, eta=0.05, max_epochs=2, mode=0, nce_k=5,
              noise_floor=1e-3, divergence_factor=1e9)
    single = dl.Trainer(dl.TrainConfig(minibatch=G * 4, **kw), params, dl.make_vocab(V), tr, va,
                        "fp32")
    single.train()
    group = dl.LocalGroup(G)
    trainers = [dl.Trainer(dl.TrainConfig(minibatch=4, **kw), params, dl.make_vocab(V), tr, va,
                           "fp32", comm=(group, G, r)) for r in range(G)]
    with ThreadPoolExecutor(G) as ex:
        list(ex.map(lambda t: t.train(), trainers))
    for t in trainers:
        assert len(t.logs) == len(single.logs)
        for a, b in zip(t.logs, single.logs):
            tol = 1e-4 if a.epoch == 1 else 1e-2
            assert a.train_loss == pytest.approx(b.train_loss, rel=tol)
            assert a.valid_ppl == pytest.approx(b.valid_ppl, rel=tol)
        # the generator advanced by the global window's draws on every rank
        assert np.array_equal(t.model.rng_state(), single.model.rng_state())
    for a, b in zip(trainers[0].params(), trainers[-1].params()):
        assert np.array_equal(a, b)  # replicas stay bit-identical


@pytest.mark.parametrize("G,precision", [(2, "fp32"), (4, "fp32"), (2, "bf16"), (4, "bf16")])
def test_dp_vocab_parallel_window_matches_global_window(orc, G, precision):
    """Data-parallel streams + vocabulary-parallel output layer
    (dl_set_vocab_shard mode 2): rank r trains streams [r*B, (r+1)*B) of the
    global window, holds W_out rows [r*V/G, (r+1)*V/G); the hidden states are
    gathered and dh reduce-scattered.  Equals one context training the global
    minibatch (fp32: summation-order tolerance), W_in / W_rec bit-identical
    across ranks."""
    import paper_1502_00512_b200 as dl
    V, H, T, B = 1024, 64, 6, 8
    Bg = G * B
    rng = np.random.default_rng(40 + G)
    params = orc.init_uniform(V, H, 23)
    x = rng.integers(0, V, (T, Bg)).astype(np.uint32)
    y = rng.integers(2, V, (T, Bg)).astype(np.uint32)
    w = (rng.random((T, Bg)) > 0.1).astype(np.uint8)
    h0 = rng.uniform(0, 1, (Bg, H)).astype(np.float32)
    scale = 1.0 / (Bg * T)
    single = dl.GpuRnn(V, H, 0, precision)
    single.set_params(*params)
    r1, hf1 = dl.bptt_run(single, dl.WindowBatch(x, y, w), h0, scale, 1.0)
    g1 = single.grads()
    assert dl.rmsprop_update(single, 0.05)
    want = single.params() + single.opt()

    group = dl.LocalGroup(G)
    ranks = []
    for r in range(G):
        m = dl.GpuRnn(V, H, 0, precision)
        m.comm_init_local(group, r)
        m.set_vocab_shard("dp")
        m.set_params(*params)
        ranks.append(m)

    def run(r):
        sl = slice(r * B, (r + 1) * B)
        wb = dl.WindowBatch(np.ascontiguousarray(x[:, sl]), np.ascontiguousarray(y[:, sl]),
                            np.ascontiguousarray(w[:, sl]))
        res, hf = dl.bptt_run(ranks[r], wb, np.ascontiguousarray(h0[sl]), scale, 1.0)
        g = ranks[r].grads()
        ok = dl.rmsprop_update(ranks[r], 0.05)
        return res, hf, g, ok

    with ThreadPoolExecutor(G) as ex:
        outs = list(ex.map(run, range(G)))
    tol = 1e-4 if precision == "fp32" else 2e-2
    for r, (res, hf, g, ok) in enumerate(outs):
        assert ok
        assert res.positions == r1.positions
        assert res.loss == pytest.approx(r1.loss, rel=1e-5 if precision == "fp32" else 1e-3)
        assert np.allclose(hf, hf1[r * B:(r + 1) * B], atol=1e-6 if precision == "fp32" else 2e-2)
    got = [m.params() + m.opt() for m in ranks]
    for r in range(1, G):  # W_in, W_rec and their state replicate bit-identically
        for k in (0, 1, 3, 4):
            assert np.array_equal(got[0][k], got[r][k])
    # the full W_out / m_out / dW_out are the rank blocks
    w_out = _assemble([got[r][2] for r in range(G)], G)
    m_out = _assemble([got[r][5] for r in range(G)], G)
    g_out = _assemble([outs[r][2][2] for r in range(G)], G)
    if precision == "fp32":
        assert close(g_out, g1[2])
        for a, b in zip(got[0][:2] + (w_out,) + got[0][3:5] + (m_out,), want):
            assert close(a, b)
    else:
        d = np.abs(w_out.astype(np.float64) - want[2])
        assert d.max() <= 2e-2 * max(1.0, np.abs(want[2]).max())
        cosv = float(np.dot(g_out.ravel(), g1[2].ravel()) /
                     (np.linalg.norm(g_out) * np.linalg.norm(g1[2]) + 1e-30))
        assert cosv > 0.99


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_dp_vocab_parallel_trainer_matches_global_minibatch(orc, precision):
    """Two ranks x minibatch 4 with the vocabulary-parallel output layer ==
    one trainer with minibatch 8 (epoch losses and validation perplexities)."""
    import paper_1502_00512_b200 as dl
    V, H, G = 96, 64, 2
    tr, va = orc.random_stream_pair(19, V, 4016, 600)
    tr = tr[:4000]
    params = orc.init_uniform(V, H, 11)
    kw = dict(nstate=H, noffset=3, unroll=5, eta=0.02, max_epochs=2, mode=1)
    single = dl.Trainer(dl.TrainConfig(minibatch=G * 4, **kw), params, dl.make_vocab(V), tr, va,
                        precision)
    single.train()
    group = dl.LocalGroup(G)
    trainers = [dl.Trainer(dl.TrainConfig(minibatch=4, **kw), params, dl.make_vocab(V), tr, va,
                           precision, comm=(group, G, r), vocab_shard="dp") for r in range(G)]
    with ThreadPoolExecutor(G) as ex:
        list(ex.map(lambda t: t.train(), trainers))
    rel = 1e-4 if precision == "fp32" else 1e-2
    for t in trainers:
        assert len(t.logs) == len(single.logs)
        for a, b in zip(t.logs, single.logs):
            assert a.train_loss == pytest.approx(b.train_loss, rel=rel)
            assert a.valid_ppl == pytest.approx(b.valid_ppl, rel=10 * rel)


@pytest.mark.parametrize("G", [2, 4])
def test_vocab_shard_bf16_repaired_rows_match_oracle(orc, G):
    """The shifted-exponential softmax across vocabulary shards when rows need
    a new shift: W_out rows that put one logit ~48 nats (rescale) and one
    ~110 nats (a half tile past the epilogue's cap, redone against its own
    maximum) above the others, on different shards.  Each rank's block lse
    after its own rescales goes through the exchange; loss and gradients
    against the fp32 oracle."""
    import paper_1502_00512_b200 as dl
    V, H, T, B = 1024, 128, 4, 16
    rng = np.random.default_rng(70 + G)
    w_in, w_rec, w_out = (rng.uniform(-0.1, 0.1, s).astype(np.float32)
                          for s in ((V, H), (H, H), (V, H)))
    w_out[5] = 0.75           # ~48 nats above the rest (first shard): rescaled
    w_out[V - 3] = 1.7        # ~110 nats (last shard): past the 2^120 cap
    params = (w_in, w_rec, w_out)
    x = rng.integers(0, V, (T, B)).astype(np.uint32)
    y = rng.integers(8, V - 8, (T, B)).astype(np.uint32)
    w = (rng.random((T, B)) > 0.1).astype(np.uint8)
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    scale = 1.0 / (B * T)
    want = orc.bptt(params, 0, x, y, w, h0, scale, 5.0)
    ranks = _vshard_ranks(dl, G, V, H, "bf16", params)
    wb = dl.WindowBatch(x, y, w)

    def run(r):
        res, hf = dl.bptt_run(ranks[r], wb, h0, scale, 5.0)
        return res, ranks[r].grads()

    with ThreadPoolExecutor(G) as ex:
        outs = list(ex.map(run, range(G)))
    for res, g in outs:
        assert res.positions == want["positions"]
        assert np.isfinite(res.loss)
        assert res.loss == pytest.approx(want["loss"], rel=2e-3)
    g_in, g_rec = outs[0][1][0], outs[0][1][1]
    for name, got, ref_ in (("dW_in", g_in, want["g_in_dense"]), ("dW_rec", g_rec, want["g_rec"])):
        assert np.all(np.isfinite(got)), name
        err = np.linalg.norm(got - ref_) / np.linalg.norm(ref_)
        assert err < 2e-2, (name, err)
    for m in ranks:
        m.close()
