"""GPU parity of the forward scorers: per-token log-probabilities of the
sharded walk (eval.hpp:151-222), sharded_perplexity, rnn_perplexity
(eval.hpp:84-145) and exact n-best rescoring (eval.hpp:693-790), fp32 mode
against the oracle (per-token logp within 1e-4 relative + 1e-5 absolute)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["fp32", "tf32x3"])
@pytest.mark.parametrize("V,H,shards,n,act", [
    (30, 8, 8, 200, 0), (200, 32, 3, 1000, 1), (1000, 64, 64, 4000, 0),
    (10000, 128, 8, 3000, 0),
])
def test_sharded_logprobs_match_oracle(orc, V, H, shards, n, act, precision):
    import paper_1502_00512_b200 as dl
    params = orc.init_uniform(V, H, 5 + V)
    ids = orc.random_stream(77 + V, V, n)[:n]
    want = orc.sharded_logprobs(params, act, ids, shards)
    m = dl.GpuRnn(V, H, act, precision)
    m.set_params(*params)
    r = dl.sharded_perplexity(m, ids, shards)
    ro = orc.sharded_ppl(params, act, ids, shards)
    assert r.predicted == ro["predicted"]
    assert r.total_logprob == pytest.approx(ro["total_logprob"], rel=1e-5)
    assert r.perplexity == pytest.approx(ro["perplexity"], rel=1e-5)
    # per-token: rebuild the lock-step inputs exactly as eval.hpp:178-195
    S = min(shards, n // 2)
    begin = [s * n // S for s in range(S + 1)]
    steps = max(begin[s + 1] - begin[s] for s in range(S)) - 1
    x = np.zeros((steps, S), np.uint32)
    t = np.full((steps, S), -1, np.int64)
    for j in range(steps):
        for s in range(S):
            if j + 1 < begin[s + 1] - begin[s]:
                x[j, s] = ids[begin[s] + j]
                yy = ids[begin[s] + j + 1]
                t[j, s] = -1 if yy == 1 else yy
    lp, tot, pred, _ = dl.score(m, x, t)
    assert np.array_equal(np.isnan(lp), np.isnan(want))
    ok = ~np.isnan(want)
    err = np.abs(lp[ok] - want[ok])
    assert np.all(err <= 1e-4 * np.abs(want[ok]) + 1e-5), err.max()


def test_rnn_perplexity_matches_oracle(orc):
    import paper_1502_00512_b200 as dl
    V, H = 500, 48
    params = orc.init_uniform(V, H, 12)
    ids = orc.random_stream(9, V, 700)
    want = orc.rnn_ppl(params, 0, ids)
    m = dl.GpuRnn(V, H, 0, "fp32")
    m.set_params(*params)
    r = dl.rnn_perplexity(m, ids)
    assert r.predicted == want["predicted"]
    assert r.perplexity == pytest.approx(want["perplexity"], rel=1e-5)


def test_scorer_errors_follow_reference(orc):
    import paper_1502_00512_b200 as dl
    m = dl.GpuRnn(10, 4, 0, "fp32")
    with pytest.raises(ValueError):
        dl.sharded_perplexity(m, np.array([3], np.uint32), 4)
    with pytest.raises(ValueError):
        dl.sharded_perplexity(m, np.array([3, 4, 5], np.uint32), 0)
    with pytest.raises(dl.DataError):
        dl.sharded_perplexity(m, np.array([3, 40, 5, 6], np.uint32), 2)
    with pytest.raises(ValueError):  # only bos targets -> nothing predicted
        dl.rnn_perplexity(m, np.array([1, 1, 1], np.uint32))


def test_rescore_matches_reference(ref):
    import paper_1502_00512_b200 as dl
    V, H = 40, 16
    params = ref.init_uniform(V, H, 3)
    words = dl.make_vocab(V)
    rng = np.random.default_rng(5)
    lines = []
    for u in range(4):
        for h in range(5):
            n = int(rng.integers(0, 7))
            ws = " ".join("oov" if rng.random() < 0.1 else words[int(rng.integers(3, V))]
                          for _ in range(n))
            ac = float(rng.normal(-100, 5))
            lines.append(f"u{u}\t{ac:.3f}\t{-20.0:.3f}" + (f"\t{ws}" if n else ""))
    text = "\n".join(lines) + "\n"
    want = ref.rescore(params, 0, text, lm_scale=0.7, wip=0.5)
    m = dl.GpuRnn(V, H, 0, "fp32")
    m.set_params(*params)
    utts = dl.read_nbest(text)
    dl.rescore_nbest(utts, m, words, lm_scale=0.7, wip=0.5)
    got = dl.write_nbest(utts)
    gl, wl = got.splitlines(), want.splitlines()
    assert len(gl) == len(wl)
    for a, b in zip(gl, wl):
        fa, fb = a.split("\t"), b.split("\t")
        assert fa[:4] == fb[:4] and fa[6] == fb[6]
        assert float(fa[4]) == pytest.approx(float(fb[4]), abs=2e-3)


def test_ln_z_samples_match_reference_fixture():
    """ln_z_samples (eval.hpp:805-857) on the device (fp32 parity mode)
    against the reference's fixture; drift_stats over them."""
    import os
    import paper_1502_00512_b200 as dl
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ln_z.npz"))
    V, H = g["w_in"].shape
    m = dl.GpuRnn(V, H, int(g["act"]), "fp32")
    m.set_params(g["w_in"], g["w_rec"], g["w_out"])
    z = dl.ln_z_samples(m, g["ids"], int(g["count"]))
    assert len(z) == len(g["ln_z"])
    np.testing.assert_allclose(z, g["ln_z"], rtol=1e-6)
    s = dl.drift_stats(z)
    assert s.contexts == int(g["stats"][5])
    assert s.median == pytest.approx(g["stats"][1], rel=1e-6)


def test_ln_z_samples_bf16_close_to_oracle(orc):
    import paper_1502_00512_b200 as dl
    V, H = 4096, 256
    params = orc.init_uniform(V, H, 21)
    ids = orc.random_stream(3, V, 20000)
    want = orc.ln_z_samples(params, 0, ids, 300)
    for precision, tol in (("fp32", 1e-6), ("bf16", 5e-3)):
        m = dl.GpuRnn(V, H, 0, precision)
        m.set_params(*params)
        z = dl.ln_z_samples(m, ids, 300)
        assert len(z) == len(want)
        np.testing.assert_allclose(z, want, rtol=tol)
