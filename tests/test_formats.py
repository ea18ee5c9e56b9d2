"""Host-side file formats (paper_1502_00512_b200/formats.py) byte-for-byte
against the reference writers: RNLM (rnn.hpp:263-308), ROPT
(rmsprop.hpp:137-170) and RTRN (trainer.hpp:274-341, config echo
:412-457), plus the reference's reader error behaviour."""
import os

import numpy as np
import pytest

import oracle
from paper_1502_00512_b200 import DataError, TrainConfig, formats, make_vocab

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_rnlm_matches_golden_and_roundtrips():
    g = np.load(os.path.join(GOLD, "train.npz"))
    params = (g["w_in"], g["w_rec"], g["w_out"])
    blob = formats.write_params(params, make_vocab(30), 0)
    assert blob == g["rnlm"].tobytes()
    (a, b, c), act, words = formats.read_params(blob)
    assert act == 0 and words == make_vocab(30)
    for u, v in zip((a, b, c), params):
        assert np.array_equal(u, v)
    with pytest.raises(DataError):
        formats.read_params(blob[:-3])
    with pytest.raises(DataError):
        formats.read_params(b"XXXX" + blob[4:])


def test_rtrn_untrained_matches_golden():
    g = np.load(os.path.join(GOLD, "train.npz"))
    params = (g["w_in"], g["w_rec"], g["w_out"])
    cfg = TrainConfig(nstate=8, noffset=2, minibatch=2, unroll=5, eta=0.05, max_epochs=3, mode=1)
    L = len(g["train"])
    N = 4
    cur = np.array([i * L // N for i in range(N)], np.int64)
    hid = np.full((N, 8), 0.5, np.float32)
    V = 30
    zero = (np.zeros((8, 8), np.float32), np.zeros(V, np.float32), np.zeros(V, np.float32))
    blob = formats.write_trainer(cfg, 0, cfg.eta, 0.0, 0, 0.0, formats.mt19937_64_text(cfg.seed),
                                 cur, hid, params, make_vocab(V), zero)
    assert blob == g["rtrn0"].tobytes()
    st = formats.read_trainer(blob, cfg, N, 8, L)
    assert np.array_equal(st["cursors"], cur)
    with pytest.raises(DataError):  # config mismatch
        formats.read_trainer(blob, TrainConfig(nstate=8, noffset=2, minibatch=2, unroll=6, mode=1), N, 8, L)
    # max_epochs may change on resume (trainer.hpp:446-447)
    formats.read_trainer(blob, TrainConfig(nstate=8, noffset=2, minibatch=2, unroll=5, eta=0.05,
                                           max_epochs=9, mode=1), N, 8, L)
    with pytest.raises(DataError):
        formats.read_trainer(blob, cfg, N + 1, 8, L)


def test_rtrn_trained_roundtrip_via_writer():
    g = np.load(os.path.join(GOLD, "train.npz"))
    cfg = TrainConfig(nstate=8, noffset=2, minibatch=2, unroll=5, eta=0.05, max_epochs=3, mode=1)
    blob = g["rtrn"].tobytes()
    st = formats.read_trainer(blob, cfg, 4, 8, len(g["train"]))
    again = formats.write_trainer(cfg, st["epoch"], st["eta"], st["best"], st["bad"],
                                  st["initial"], st["rng_text"], st["cursors"], st["hidden"],
                                  st["params"], st["vocab"], st["opt"])
    assert again == blob


def test_ropt_matches_reference(ref):
    rng = np.random.default_rng(163)
    V, H = 7, 3
    st = (rng.random((H, H)).astype(np.float32), rng.random(V).astype(np.float32),
          rng.random(V).astype(np.float32))
    blob = formats.write_rmsprop(V, H, 0.9, 1e-5, st)
    assert blob == ref.write_rmsprop(V, H, 0.9, 1e-5, st)
    assert len(blob) == formats.RMSPROP_HEADER_BYTES + (H * H + 2 * V) * 4
    V2, H2, rho, eps, st2 = formats.read_rmsprop(blob)
    assert (V2, H2, rho, eps) == (V, H, 0.9, 1e-5)
    for a, b in zip(st, st2):
        assert np.array_equal(a, b)
    with pytest.raises(DataError):
        formats.read_rmsprop(blob[:-3])


def test_rng_text_matches_reference(ref):
    """The RTRN generator text (trainer.hpp:283-285) for several seeds."""
    V, H = 10, 4
    for seed in (1, 7, 123456789):
        cfg = oracle.TrainConfig(nstate=H, noffset=1, minibatch=1, unroll=2, mode=1, seed=seed)
        tr = ref.random_stream(3, V, 50)
        blob, _, _ = ref.train(cfg, ref.init_uniform(V, H, 1), tr, tr, run=False)
        pcfg = TrainConfig(nstate=H, noffset=1, minibatch=1, unroll=2, seed=seed, mode=1)
        st = formats.read_trainer(blob, pcfg, 1, H, len(tr))
        assert st["rng_text"] == formats.mt19937_64_text(seed)


def test_init_uniform_is_bit_identical_to_reference():
    """dl_init_uniform (host C ABI) vs the reference's init_uniform fixture."""
    import paper_1502_00512_b200 as dl
    g = np.load(os.path.join(GOLD, "kat.npz"))
    got = np.concatenate([a.ravel()[:16] for a in dl.init_uniform(7, 5, 11)])
    assert np.array_equal(got, g["init_11"])
    t = np.load(os.path.join(GOLD, "train.npz"))
    for a, b in zip(dl.init_uniform(30, 8, 3), (t["w_in"], t["w_rec"], t["w_out"])):
        assert np.array_equal(a, b)


def test_id_stream_and_vocab_text_formats():
    words = make_vocab(6)
    assert formats.read_vocab(formats.write_vocab(words)) == words
    with pytest.raises(DataError):
        formats.read_vocab("a\nb\nc\n")
    ids = np.array([1, 4, 3, 2, 1, 5, 2], np.uint32)
    text = formats.write_id_stream(ids)
    assert text == "1 4 3 2\n1 5 2\n"
    assert np.array_equal(formats.read_id_stream(text, 6), ids)
    with pytest.raises(DataError):
        formats.read_id_stream("1 9 2", 6)
    with pytest.raises(DataError):
        formats.read_id_stream("1 x 2", 6)
