"""Scorers that combine the device RNN with host n-gram logic (SURVEY.md §8f
row 3): interpolation with a backoff model and the shortlist hit rate.  The
recurrent side of each runs on the B200 (``dl_score`` for per-token
log-probabilities, ``dl_score_candidates`` for raw candidate scores); the
n-gram side is ``ngram.NGramModel`` on the host.

==============================  ==============================================
this module                     reference (include/desklm/eval.hpp)
==============================  ==============================================
``VocabMap`` / ``make_vocab_map``  ``VocabMap`` / ``make_vocab_map`` (:231-262)
``interpolation_terms``         ``interpolation_terms`` (:297-405)
``interp_perplexity_at``        ``interp_perplexity_at`` (:407-422)
``tune_lambda``                 ``tune_lambda`` (:424-450), golden section
``interpolated_perplexity``     ``interpolated_perplexity`` (:452-461)
``hit_rate``, ``RnnHitScorer``, ``hit_rate`` (:544-592), ``RnnHitScorer``
``NgramHitScorer``              (:476-510), ``NgramHitScorer`` (:512-542)
==============================  ==============================================
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from ._lib import DataError, load


@dataclass
class VocabMap:
    full_to_rnn: List[int]
    rnn_to_full: List[int]
    oor_ids: List[int]
    rnn_unk: int = 0


def make_vocab_map(rnn_words: Sequence[str], full_words: Sequence[str], unk_id: int = 0) -> VocabMap:
    """eval.hpp:238-262: every RNN word must exist in the n-gram vocabulary;
    out-of-range ids are the unmapped n-gram words plus unk."""
    index = {w: i for i, w in enumerate(full_words)}
    full_to_rnn = [-1] * len(full_words)
    rnn_to_full = [0] * len(rnn_words)
    for r, w in enumerate(rnn_words):
        if w not in index:
            raise DataError(f"vocabulary map: word '{w}' missing from the n-gram vocabulary")
        f = index[w]
        rnn_to_full[r] = f
        full_to_rnn[f] = r
    oor = [f for f in range(len(full_words)) if full_to_rnn[f] < 0 or f == unk_id]
    return VocabMap(full_to_rnn, rnn_to_full, oor, unk_id)


@dataclass
class InterpTerm:
    a: float
    b: float


def interpolation_terms(rnn, vmap: VocabMap, ngram, ids, bos_id: int = 1) -> List[InterpTerm]:
    """Both models over the stream once (eval.hpp:297-405): per predicted
    position a = p_rnn(target) (or p_rnn(unk) * p_ng(target) / Z_out for an
    unmapped target), b = p_ng(target).  The RNN walks the stream on the
    device (one lock-step stream, dl_score); the n-gram context on the host."""
    from . import score
    ids = [int(x) for x in ids]
    if len(ids) < 2:
        raise ValueError("interpolation: stream too short")
    if len(vmap.full_to_rnn) != ngram.V:
        raise ValueError("interpolation: map/vocabulary mismatch")
    if len(vmap.rnn_to_full) != rnn.V:
        raise ValueError("interpolation: map/model mismatch")
    n = len(ids) - 1
    x_rnn = np.empty((n, 1), np.uint32)
    tgt = np.full((n, 1), -1, np.int64)
    pend = []
    ctx: List[int] = []
    maxc = ngram.order() - 1
    for i in range(n):
        x = ids[i]
        if x >= ngram.V:
            raise DataError("interpolation: id out of vocabulary range")
        xr = vmap.full_to_rnn[x]
        x_rnn[i, 0] = xr if xr >= 0 else vmap.rnn_unk
        if x == bos_id:
            ctx = [x]
        else:
            ctx.append(x)
            if maxc > 0 and len(ctx) > maxc:
                ctx = ctx[len(ctx) - maxc:]
        y = ids[i + 1]
        if y == bos_id:
            continue
        pn = math.exp(ngram.logprob(ctx, y))
        yr = vmap.full_to_rnn[y]
        if yr >= 0 and yr != vmap.rnn_unk:
            tgt[i, 0] = yr
            pend.append((i, pn, None))
        else:
            tgt[i, 0] = vmap.rnn_unk
            z_out = 0.0
            for f in vmap.oor_ids:
                z_out += math.exp(ngram.logprob(ctx, f))
            pend.append((i, pn, z_out))
    if not pend:
        raise ValueError("interpolation: no predicted tokens")
    lp, _, _, _ = score(rnn, x_rnn, tgt)
    terms = []
    for i, pn, z_out in pend:
        p = math.exp(lp[i, 0])
        if z_out is None:
            terms.append(InterpTerm(p, pn))
        else:
            terms.append(InterpTerm(p * pn / z_out if z_out > 0.0 else 0.0, pn))
    return terms


def interp_perplexity_at(terms: Sequence[InterpTerm], lam: float):
    """eval.hpp:407-422 -> (perplexity, total ln p, predicted)."""
    if not terms:
        raise ValueError("interpolation: no cached terms")
    total = 0.0
    for t in terms:
        p = lam * t.a + (1.0 - lam) * t.b
        if not p > 0.0:
            raise DataError("interpolation: non-positive mixture")
        total += math.log(p)
    return math.exp(-total / len(terms)), total, len(terms)


def tune_lambda(terms: Sequence[InterpTerm]):
    """Golden-section search over lambda in [0, 1] (eval.hpp:424-450) ->
    (lambda, best perplexity)."""
    inv_phi = 0.6180339887498949
    lo, hi = 0.0, 1.0
    x1, x2 = hi - inv_phi * (hi - lo), lo + inv_phi * (hi - lo)
    f1, f2 = interp_perplexity_at(terms, x1)[0], interp_perplexity_at(terms, x2)[0]
    it = 0
    while it < 120 and hi - lo > 1e-10:
        if f1 <= f2:
            hi, x2, f2 = x2, x1, f1
            x1 = hi - inv_phi * (hi - lo)
            f1 = interp_perplexity_at(terms, x1)[0]
        else:
            lo, x1, f1 = x1, x2, f2
            x2 = lo + inv_phi * (hi - lo)
            f2 = interp_perplexity_at(terms, x2)[0]
        it += 1
    lam = 0.5 * (lo + hi)
    return lam, interp_perplexity_at(terms, lam)[0]


def interpolated_perplexity(rnn, vmap, ngram, ids, lam: float):
    return interp_perplexity_at(interpolation_terms(rnn, vmap, ngram, ids), lam)


# ----------------------------------------------------------------- hit rate
class NgramHitScorer:
    """eval.hpp:512-542: candidates scored by the n-gram log-probability."""

    def __init__(self, model, bos_id: int = 1):
        self.model, self.bos = model, bos_id

    def score_all(self, ids, cands):
        out, ctx = [], []
        cap = self.model.order() - 1
        for x, cl in zip(ids, cands):
            if x == self.bos:
                ctx = [x]
            else:
                ctx.append(x)
                if cap > 0 and len(ctx) > cap:
                    ctx = ctx[len(ctx) - cap:]
            out.append([self.model.logprob(ctx, w) for w in cl])
        return out


class RnnHitScorer:
    """eval.hpp:476-510: candidates scored by the recurrent model's raw
    output scores, computed on the device for the whole stream at once
    (dl_score_candidates)."""

    def __init__(self, model):
        self.model = model

    def score_all(self, ids, cands):
        steps = len(ids)
        K = max(1, max((len(c) for c in cands), default=1))
        cand = np.full((steps, K), -1, np.int64)
        for j, cl in enumerate(cands):
            cand[j, :len(cl)] = cl
        x = np.ascontiguousarray(ids, np.uint32)
        out = np.zeros((steps, K), np.float32)
        self.model._chk(load().dl_score_candidates(self.model.handle, x.ctypes.data, steps, K,
                                                   cand.ctypes.data, out.ctypes.data))
        return [[float(out[j, k]) for k in range(len(cl))] for j, cl in enumerate(cands)]


def hit_rate(ids, shortlist_model, shortlist_k: int, top_k: int, scorer, bos_id: int = 1):
    """Fraction of predicted positions whose target is in the top_k of the
    shortlist after reranking by the scorer (eval.hpp:544-592); ties break
    toward the smaller id -> (positions, hits)."""
    if top_k < 1 or shortlist_k < top_k:
        raise ValueError("hit rate: need 1 <= top_k <= shortlist_k")
    ids = [int(x) for x in ids]
    if len(ids) < 2:
        raise ValueError("hit rate: stream too short")
    cap = shortlist_model.order() - 1
    ctx: List[int] = []
    lists, targets, keep = [], [], []
    for i in range(len(ids) - 1):
        x = ids[i]
        if x == bos_id:
            ctx = [x]
        else:
            ctx.append(x)
            if cap > 0 and len(ctx) > cap:
                ctx = ctx[len(ctx) - cap:]
        y = ids[i + 1]
        if y == bos_id:
            lists.append([])
            targets.append(-1)
            continue
        sl = shortlist_model.shortlist(ctx, shortlist_k)
        targets.append(y)
        lists.append(sl if y in sl else [])
        keep.append(i)
    positions = len(keep)
    if positions == 0:
        raise ValueError("hit rate: no predicted tokens")
    scores = scorer.score_all(ids[:-1], lists)
    hits = 0
    for i in keep:
        sl = lists[i]
        if not sl:
            continue
        ranked = sorted(zip((-s for s in scores[i]), sl))
        if targets[i] in [w for _, w in ranked[:min(top_k, len(ranked))]]:
            hits += 1
    return positions, hits
