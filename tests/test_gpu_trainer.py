"""GPU parity of the device-resident Trainer (trainer.hpp:171-476): the
offset-stream schedule (cursors, window arrays, wrap resets) must be
bit-exact; losses / perplexities within 1e-4 (fp32 mode); the RTRN
checkpoint must round-trip and resume must equal an uninterrupted run."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def make_data(orc, V, L, nvalid, seed):
    tr, va = orc.random_stream_pair(seed, V, L + 16, nvalid)
    return tr[:L], va


@pytest.mark.parametrize("H,noffset,B,T,L,act", [
    (8, 2, 2, 5, 400, 0), (16, 3, 2, 4, 999, 1), (32, 4, 8, 8, 3000, 0),
])
def test_epochs_match_oracle(orc, H, noffset, B, T, L, act):
    import paper_1502_00512_b200 as dl
    V = 60
    tr, va = make_data(orc, V, L, 300, 1000 + H)
    params = orc.init_uniform(V, H, 7 + H)
    kw = dict(nstate=H, noffset=noffset, minibatch=B, unroll=T, eta=0.05, max_epochs=3,
              mode=1, act=act)
    t = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, "fp32")
    try:
        want = orc.train(oracle.TrainConfig(**kw), params, tr, va)
    except oracle.OracleError as e:
        assert e.code == 2  # the reference diverges (DataError, trainer.hpp:258-261)
        with pytest.raises(dl.DataError):
            t.train()
        return
    t.train()
    assert len(t.logs) == len(want["logs"])
    assert t.initial_ppl == pytest.approx(want["initial_ppl"], rel=1e-5)
    # one-step numbers agree to 1e-4; fp32 rounding differences then compound
    # chaotically over hundreds of rmsprop steps, so later epochs get the
    # north star's N-step bar (validation perplexity within 1%)
    for lg, w in zip(t.logs, want["logs"]):
        tol = 1e-4 if lg.epoch == 1 else 1e-2
        assert lg.epoch == int(w[0])
        assert lg.train_loss == pytest.approx(w[1], rel=tol)
        assert lg.valid_ppl == pytest.approx(w[2], rel=tol)
        assert lg.eta == w[3]
        assert lg.skipped_updates == int(w[6])
    cur, hid = t.model.trainer_state()
    assert np.array_equal(cur, want["cursors"])  # bit-exact schedule
    if len(t.logs) == 1:  # carried hidden state: compared while still one-step close
        assert np.abs(hid - want["hidden"]).max() <= 1e-3 * np.abs(want["hidden"]).max() + 1e-6


def test_frozen_weights_replay_exactly(orc):
    """test_trainer.cpp:253-282: eta = 1e-15 freezes the weights, so the
    epoch loss is a pure function of the schedule."""
    import paper_1502_00512_b200 as dl
    V, H = 40, 8
    tr, va = make_data(orc, V, 777, 200, 31)
    params = orc.init_uniform(V, H, 3)
    kw = dict(nstate=H, noffset=2, minibatch=2, unroll=5, eta=1e-15, max_epochs=1, mode=1)
    want = orc.train(oracle.TrainConfig(**kw), params, tr, va)
    t = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, "fp32")
    t.train()
    for a, b in zip(t.params(), params):
        assert np.array_equal(a, b)
    assert t.logs[0].train_loss == pytest.approx(want["logs"][0][1], rel=1e-5)
    cur, _ = t.model.trainer_state()
    assert np.array_equal(cur, want["cursors"])


def test_checkpoint_resume_is_bit_exact(orc):
    """test_trainer.cpp:498-551: resume after 2 epochs == straight 3."""
    import paper_1502_00512_b200 as dl
    V, H = 50, 16
    tr, va = make_data(orc, V, 1200, 300, 44)
    params = orc.init_uniform(V, H, 9)
    kw = dict(nstate=H, noffset=2, minibatch=4, unroll=6, eta=0.05, max_epochs=3, mode=1)
    straight = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, "fp32")
    straight.train()
    kw2 = dict(kw, max_epochs=2)
    a = dl.Trainer(dl.TrainConfig(**kw2), params, dl.make_vocab(V), tr, va, "fp32")
    a.train()
    blob = a.save_checkpoint()
    b = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, "fp32")
    b.load_checkpoint(blob)
    assert b.save_checkpoint()[:64] == blob[:64]
    b.train()
    assert b.epoch == straight.epoch
    assert b.save_checkpoint() == straight.save_checkpoint()


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_resume_then_several_epochs_is_bit_exact(orc, precision):
    """Resume followed by two more epochs: after load_checkpoint
    train() skips the initial validation, so the first epoch's window graphs
    are captured before validate() grows the workspace; the next epoch must
    re-capture rather than replay graphs holding freed buffers."""
    import paper_1502_00512_b200 as dl
    V, H = 64, 16
    tr, va = make_data(orc, V, 1500, 400, 45)
    params = orc.init_uniform(V, H, 19)
    kw = dict(nstate=H, noffset=2, minibatch=8, unroll=6, eta=0.05, max_epochs=4, mode=1)
    straight = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, precision)
    straight.train()
    a = dl.Trainer(dl.TrainConfig(**dict(kw, max_epochs=2)), params, dl.make_vocab(V), tr, va,
                   precision)
    a.train()
    b = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, precision)
    b.load_checkpoint(a.save_checkpoint())
    b.train()
    assert b.epoch == straight.epoch >= 3
    assert [l.train_loss for l in b.logs] == [l.train_loss for l in straight.logs[2:]]
    assert b.save_checkpoint() == straight.save_checkpoint()


def test_scoring_between_trainer_runs(orc):
    """dl_score / sharded_perplexity with a larger bank between two
    dl_trainer_run calls reallocates the window workspace: the trainer's
    cached graphs must be dropped (identical to running without scoring)."""
    import paper_1502_00512_b200 as dl
    V, H = 80, 32
    tr, va = make_data(orc, V, 2000, 3000, 46)
    params = orc.init_uniform(V, H, 23)
    runs = []
    for interleave in (False, True):
        m = dl.GpuRnn(V, H, 0, "bf16")
        m.set_params(*params)
        m.set_opt(None, None, None, 0.9995, 1e-6)
        m.trainer_init(tr, 2, 8, 5, 1.0)
        l1, _ = m.trainer_run(0, 6, 0.05)
        if interleave:
            dl.sharded_perplexity(m, va, 16)   # grows the window buffers
            dl.sharded_perplexity(m, va, 64)
        l2, _ = m.trainer_run(6, 6, 0.05)
        runs.append((l1, l2, m.params(), m.trainer_state()))
        m.close()
    (a1, a2, pa, sa), (b1, b2, pb, sb) = runs
    assert a1 == b1 and a2 == b2
    for x, y in zip(pa + sa, pb + sb):
        assert np.array_equal(x, y)


def test_checkpoint_layout_matches_reference(orc, ref):
    """Untrained trainer: the RTRN bytes equal the reference's exactly."""
    import paper_1502_00512_b200 as dl
    V, H = 30, 8
    tr, va = make_data(orc, V, 400, 120, 77)
    params = orc.init_uniform(V, H, 3)
    kw = dict(nstate=H, noffset=2, minibatch=2, unroll=5, eta=0.05, max_epochs=3, mode=1)
    blob, _, _ = ref.train(oracle.TrainConfig(**kw), params, tr, va, run=False)
    t = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr, va, "fp32")
    assert t.save_checkpoint() == blob


def test_trainer_rejects_bad_setups(orc):
    import paper_1502_00512_b200 as dl
    V, H = 20, 4
    tr, va = make_data(orc, V, 100, 50, 1)
    params = orc.init_uniform(V, H, 3)
    with pytest.raises(ValueError):
        dl.Trainer(dl.TrainConfig(nstate=H, noffset=64, minibatch=8, mode=1), params,
                   dl.make_vocab(V), tr, va)
    with pytest.raises(ValueError):
        dl.Trainer(dl.TrainConfig(nstate=H, noffset=2, minibatch=2, mode=1), params,
                   dl.make_vocab(V - 1), tr, va)
    with pytest.raises(ValueError):
        dl.Trainer(dl.TrainConfig(nstate=H, noffset=2, minibatch=2, mode=1), params,
                   dl.make_vocab(V), tr, va[:1])
