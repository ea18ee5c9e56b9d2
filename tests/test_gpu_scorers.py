"""GPU side of the interpolation and hit-rate scorers:
the recurrent model's per-token probabilities (dl_score) and raw candidate
scores (dl_score_candidates) combined with the host n-gram model, against
the reference's own interpolation_terms / tune_lambda / hit_rate
(tests/golden/ngram_scorers.npz)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "ngram_scorers.npz"))


def test_interpolation_terms_match_reference(g):
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import ngram, scorers
    Vf, Vr, H = int(g["Vf"]), int(g["Vr"]), int(g["H"])
    m = ngram.estimate_kn(ngram.count_ngrams(g["train"], int(g["order"])), Vf)
    rnn = dl.GpuRnn(Vr, H, 0, "fp32")
    rnn.set_params(g["w_in"], g["w_rec"], g["w_out"])
    vmap = scorers.make_vocab_map(dl.make_vocab(Vr), dl.make_vocab(Vf))
    terms = scorers.interpolation_terms(rnn, vmap, m, g["eval"])
    assert len(terms) == len(g["interp_a"])
    np.testing.assert_allclose([t.a for t in terms], g["interp_a"], rtol=1e-5)
    np.testing.assert_allclose([t.b for t in terms], g["interp_b"], rtol=1e-12)
    lam, ppl = scorers.tune_lambda(terms)
    assert lam == pytest.approx(float(g["interp_lambda"]), abs=1e-4)
    assert ppl == pytest.approx(float(g["interp_ppl"]), rel=1e-5)


def test_rnn_hit_rate_matches_reference(g):
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import ngram, scorers
    Vf, H = int(g["Vf"]), int(g["H"])
    m = ngram.estimate_kn(ngram.count_ngrams(g["train"], int(g["order"])), Vf)
    rnn = dl.GpuRnn(Vf, H, 0, "fp32")
    rnn.set_params(g["hw_in"], g["hw_rec"], g["hw_out"])
    for sk, tk, kind, pos, hits in g["hits"]:
        if kind != 0:
            continue
        got = scorers.hit_rate(g["eval"], m, int(sk), int(tk), scorers.RnnHitScorer(rnn))
        assert got[0] == int(pos)
        # raw scores are the reference's 8-lane double dot products; only a
        # recurrence rounding difference at an exact score tie could move a hit
        assert abs(got[1] - int(hits)) <= 1


def test_candidate_scores_are_reference_dot_products(orc):
    """dl_score_candidates == float(dot_acc(h, W_out[w])) of the oracle's
    single-stream states (fp32 mode)."""
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import scorers
    V, H = 300, 32
    params = orc.init_uniform(V, H, 8)
    ids = orc.random_stream(4, V, 200)[:150]
    rng = np.random.default_rng(0)
    cands = [list(rng.integers(0, V, rng.integers(0, 6))) for _ in ids]
    rnn = dl.GpuRnn(V, H, 1, "fp32")
    rnn.set_params(*params)
    got = scorers.RnnHitScorer(rnn).score_all(list(ids), cands)
    # the oracle's log-probs give s_w - lse; differences of two candidates at
    # the same position are score differences
    for j, cl in enumerate(cands):
        if len(cl) < 2:
            continue
        x = np.ascontiguousarray(ids[: j + 1], np.uint32).reshape(-1, 1)
        lps = []
        for w in cl[:2]:
            t = np.full((j + 1, 1), -1, np.int64)
            t[j, 0] = w
            lp, _, _, _ = dl.score(rnn, x, t)
            lps.append(lp[j, 0])
        assert (got[j][0] - got[j][1]) == pytest.approx(lps[0] - lps[1], abs=1e-4)
        if j > 40:
            break
