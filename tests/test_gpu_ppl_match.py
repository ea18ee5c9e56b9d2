"""PPL match at the C1 configuration (and at H = 1,024): the reference's
own PPL-match corpus (TextGenerator(GenConfig{}, 555), normalized, 10,000-word
vocabulary, first 262,144 training ids, 50,000 validation ids), init_uniform
seed 1, H=128, T=8, B=8, noffset=128 (N=1,024 streams), softmax, eta 0.05:
validation perplexity after one epoch (4,096 windows) of the device trainer
within 1% of the reference CPU trainer's (tests/golden/ppl_match_c1.npz, made
by the compiled reference, 283 s on 8 host threads)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


# One epoch at these settings is chaotic: a single run of ANY precision lands
# a few percent from the reference -- over the init seeds 1..5 the fp32 mode
# is +0.12, -3.68, +1.10, +0.49, +0.37% at C1 (scripts/ppl_seeds_c1.py; the
# reference itself moves +0.22% under a one-ulp W_rec perturbation).  The
# north star's 1% bar is therefore held per run where a single run meets it
# (fp32 at seed 1, with its training loss) and on the seed mean
# (test_ppl_match_seed_mean below: bf16 with the fp32-class modes as control).
@pytest.mark.parametrize("fixture,precision,rel", [
    ("ppl_match_c1.npz", "fp32", 1e-2),
    # H = 1,024 (K = 1,024 contractions in the recurrence and logits,
    # K = 10,000 in dh): tests/golden/make_golden.py write_ppl_match_h1024
    ("ppl_match_h1024.npz", "fp32", 1e-2)])
def test_ppl_match_one_epoch(fixture, precision, rel):
    import paper_1502_00512_b200 as dl
    g = np.load(os.path.join(GOLD, fixture))
    V, H = int(g["V"]), int(g["H"])
    params = dl.init_uniform(V, H, int(g["init_seed"]))
    cfg = dl.TrainConfig(nstate=H, noffset=128, minibatch=8, unroll=8, eta=float(g["eta"]),
                         max_epochs=1, mode=1)
    t = dl.Trainer(cfg, params, dl.make_vocab(V), g["train"], g["valid"], precision)
    t.train()
    assert t.initial_ppl == pytest.approx(float(g["initial"]), rel=1e-3)
    assert len(t.logs) == 1
    assert t.logs[0].valid_ppl == pytest.approx(float(g["logs"][0][2]), rel=rel)
    assert t.logs[0].train_loss == pytest.approx(float(g["logs"][0][1]), rel=rel)


@pytest.mark.parametrize("fixture,precision,mean_bar,max_bar", [
    # C1 (eta 0.05, seeds 1-10): fp32 -0.08%, bf16 -0.91% on the mean; a
    # single seed lands up to 3.7% (fp32) / 5.6% (bf16) away
    ("ppl_match_c1", "bf16", 1e-2, 1e-1), ("ppl_match_c1", "fp32", 1e-2, 5e-2),
    # H = 1,024, eta 0.01: the fp32-class modes stay within 0.6% on every
    # seed, the bf16 trainer within 2.8% (mean -0.44%; round 1's in-place
    # softmax path: +5.1% on the mean, +11% on seed 3 -- scripts/ppl_seeds_c1.py)
    ("ppl_match_h1024", "bf16", 1e-2, 6e-2), ("ppl_match_h1024", "fp32", 1e-2, 1e-2),
    ("ppl_match_h1024", "tf32x3", 1e-2, 1e-2)])
def test_ppl_match_seed_mean(fixture, precision, mean_bar, max_bar):
    """PPL match on the seed mean: one epoch from each init_uniform seed of
    the fixture (<fixture>.npz: seed 1; <fixture>_seeds.npz: seeds 2.., all
    from the compiled reference trainer), validation perplexity vs the
    reference's: the mean deviation within mean_bar, every seed within
    max_bar."""
    import paper_1502_00512_b200 as dl
    g = np.load(os.path.join(GOLD, fixture + ".npz"))
    sd = np.load(os.path.join(GOLD, fixture + "_seeds.npz"))
    V, H = int(g["V"]), int(g["H"])
    seeds = [int(g["init_seed"])] + [int(x) for x in sd["seeds"]]
    refs = [float(g["logs"][0][2])] + [float(l[2]) for l in sd["logs"]]
    inis = [float(g["initial"])] + [float(x) for x in sd["initial"]]
    dev = []
    for seed, ref_ppl, ini in zip(seeds, refs, inis):
        cfg = dl.TrainConfig(nstate=H, noffset=128, minibatch=8, unroll=8, eta=float(g["eta"]),
                             max_epochs=1, mode=1)
        t = dl.Trainer(cfg, dl.init_uniform(V, H, seed), dl.make_vocab(V), g["train"],
                       g["valid"], precision)
        t.train()
        assert t.initial_ppl == pytest.approx(ini, rel=1e-3)
        dev.append(t.logs[0].valid_ppl / ref_ppl - 1)
        t.model.close()
    dev = np.array(dev)
    assert abs(dev.mean()) <= mean_bar, dev
    assert np.all(np.abs(dev) <= max_bar), dev
