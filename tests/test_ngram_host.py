"""Host n-gram side of the §8f row 3 scorers (no GPU): count_ngrams +
modified Kneser-Ney estimation, backoff log-probabilities, shortlists,
n-gram perplexity, and the n-gram-scored hit rate, against the reference's
fixture (tests/golden/ngram_scorers.npz, made by oracle/_ref)."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLD, "ngram_scorers.npz"))


@pytest.mark.parametrize("order", [1, 2, 3, 4])
def test_kn_model_matches_reference(g, order):
    from paper_1502_00512_b200 import ngram
    m = ngram.estimate_kn(ngram.count_ngrams(g["train"], order), int(g["Vf"]))
    ctx = [[int(x) for x in row if x >= 0] for row in g["ctx"]]
    lp = np.array([m.logprob(c, int(w)) for c, w in zip(ctx, g["words"])])
    # (sums over hash-map levels: the reference's unordered_map order vs
    # Python's dict order -> double rounding only)
    np.testing.assert_allclose(lp, g[f"logp_{order}"], rtol=1e-12)
    for c, want in zip(ctx, g[f"shortlist_{order}"]):
        assert m.shortlist(c, 12) == [int(x) for x in want if x >= 0]
    tot, pred, ppl = ngram.ngram_perplexity_full(m, g["eval"])
    assert pred == int(g[f"ppl_{order}"][1])
    assert tot == pytest.approx(g[f"ppl_{order}"][0], rel=1e-12)


def test_ngram_hit_rate_matches_reference(g):
    from paper_1502_00512_b200 import ngram, scorers
    m = ngram.estimate_kn(ngram.count_ngrams(g["train"], int(g["order"])), int(g["Vf"]))
    for sk, tk, kind, pos, hits in g["hits"]:
        if kind != 1:
            continue
        assert scorers.hit_rate(g["eval"], m, int(sk), int(tk), scorers.NgramHitScorer(m)) == \
            (int(pos), int(hits))


def test_tune_lambda_and_mixture_on_reference_terms(g):
    """interp_perplexity_at / tune_lambda (eval.hpp:407-450) over the
    reference's own cached terms reproduce its lambda and perplexity."""
    from paper_1502_00512_b200 import scorers
    terms = [scorers.InterpTerm(float(a), float(b)) for a, b in zip(g["interp_a"], g["interp_b"])]
    lam, ppl = scorers.tune_lambda(terms)
    assert lam == pytest.approx(float(g["interp_lambda"]), abs=1e-9)
    assert ppl == pytest.approx(float(g["interp_ppl"]), rel=1e-12)
    with pytest.raises(ValueError):
        scorers.interp_perplexity_at([], 0.5)


def test_vocab_map_rules():
    from paper_1502_00512_b200 import DataError, make_vocab, scorers
    m = scorers.make_vocab_map(make_vocab(5), make_vocab(8))
    assert m.full_to_rnn == [0, 1, 2, 3, 4, -1, -1, -1]
    assert m.oor_ids == [0, 5, 6, 7]  # unk + the unmapped words
    with pytest.raises(DataError):
        scorers.make_vocab_map(make_vocab(5) + ["zz"], make_vocab(8))
