"""Backoff n-gram model on the host: the n-gram side of the interpolation and
shortlist hit-rate scorers.  The recurrent side of those
scorers runs on the device (``scorers.py``); this module restates the
reference's estimator and queries so that both sides meet in one process.

==============================  ==============================================
this module                     reference (include/desklm/ngram.hpp)
==============================  ==============================================
``count_ngrams``                ``count_ngrams`` (:97-123): windows within
                                [bos .. eos], suffixes of the longest window
``adjust_counts``               ``adjust_counts`` (:311-328): continuation
                                counts, bos-initial grams keep raw counts
``estimate_discounts``          ``detail::estimate_discounts`` (:283-304)
``estimate_kn``                 ``estimate_kn`` (:336-426): interpolated
                                modified Kneser-Ney, backoff weights = the
                                interpolation weights
``NGramModel``                  ``NGramModel`` (:138-268): log10 storage,
                                ``logprob`` (natural log) via the backoff
                                chain, exact ``shortlist``
``ngram_perplexity_full``       ``ngram_perplexity_full`` (:453-460)
==============================  ==============================================

Keys are tuples of word ids.  Sums over a level follow Python's dict order
where the reference iterates an unordered_map, so probabilities agree to
double rounding (1e-12 relative), not bit for bit.
"""
from __future__ import annotations

import math
from bisect import bisect_left
from typing import Dict, List, Sequence, Tuple

from ._lib import DataError

LOG10_BOS_PROB = -99.0  # ngram.hpp:132
_LN10 = 2.302585092994045684


def count_ngrams(ids: Sequence[int], order: int, bos_id: int = 1) -> List[Dict[tuple, int]]:
    """levels[k-1]: k-gram -> count (ngram.hpp:97-123)."""
    if order < 1:
        raise ValueError("count_ngrams: order must be >= 1")
    levels: List[Dict[tuple, int]] = [dict() for _ in range(order)]
    ids = [int(x) for x in ids]
    sent_start = 0
    for i, w in enumerate(ids):
        if w == bos_id:
            sent_start = i
        max_k = min(order, i - sent_start + 1)
        window = tuple(ids[i + 1 - max_k:i + 1])
        for k in range(max_k, 0, -1):
            lv = levels[k - 1]
            lv[window] = lv.get(window, 0) + 1
            window = window[1:]
    return levels


def adjust_counts(raw: List[Dict[tuple, int]], bos_id: int = 1) -> List[Dict[tuple, int]]:
    """Continuation-adjusted counts (ngram.hpp:311-328)."""
    order = len(raw)
    adj: List[Dict[tuple, int]] = [dict() for _ in range(order)]
    adj[order - 1] = dict(raw[order - 1])
    for k in range(order - 1, 0, -1):
        out = adj[k - 1]
        for key in adj[k]:
            s = key[1:]
            out[s] = out.get(s, 0) + 1
        for key, c in raw[k - 1].items():
            if key[0] == bos_id:
                out[key] = c
    return adj


class Discounts:
    def __init__(self, d1=0.75, d2=0.75, d3=0.75):
        self.d1, self.d2, self.d3 = d1, d2, d3

    def of(self, c: int) -> float:
        if c == 0:
            return 0.0
        if c == 1:
            return self.d1
        if c == 2:
            return self.d2
        return self.d3


def estimate_discounts(n: Sequence[int]) -> Discounts:
    """Modified KN discounts from count-of-counts n[1..4] (ngram.hpp:283-304);
    degenerate statistics fall back to 0.75."""
    if n[1] == 0 or n[2] == 0 or n[3] == 0 or n[4] == 0:
        return Discounts()
    y = n[1] / (n[1] + 2.0 * n[2])
    d = Discounts(1.0 - 2.0 * y * n[2] / n[1], 2.0 - 3.0 * y * n[3] / n[2],
                  3.0 - 4.0 * y * n[4] / n[3])
    if not (0.0 < d.d1 <= 1.0) or not (0.0 < d.d2 <= 2.0) or not (0.0 < d.d3 <= 3.0):
        return Discounts()
    return d


class NGramModel:
    """Backoff model over word ids 0..V-1: levels[k-1][k-gram] =
    [logp10, bow10, has_bow] (ngram.hpp:138-268)."""

    def __init__(self, order: int, vocab_size: int, bos_id: int = 1):
        if order < 1:
            raise ValueError("NGramModel: order must be >= 1")
        self._order, self.V, self.bos_id = order, vocab_size, bos_id
        self.levels: List[Dict[tuple, list]] = [dict() for _ in range(order)]
        self._succ: List[Dict[tuple, List[int]]] = []
        self._unigram_desc: List[int] = []

    def order(self) -> int:
        return self._order

    def find(self, key: tuple):
        if len(key) == 0 or len(key) > self._order:
            return None
        return self.levels[len(key) - 1].get(key)

    def finalize(self):
        """Successor lists and the unigram ranking (ngram.hpp:165-186)."""
        self._succ = [dict() for _ in range(max(0, self._order - 1))]
        for k in range(2, self._order + 1):
            succ = self._succ[k - 2]
            for key in self.levels[k - 1]:
                succ.setdefault(key[:-1], []).append(key[-1])
            for ws in succ.values():
                ws.sort()
        up = [-math.inf] * self.V
        for w in range(self.V):
            e = self.find((w,))
            if e is not None:
                up[w] = e[0]
        self._unigram_desc = sorted(range(self.V), key=lambda w: (-up[w], w))

    def logprob(self, context: Sequence[int], word: int) -> float:
        """Natural-log probability via the backoff chain (ngram.hpp:190-208)."""
        if word >= self.V:
            raise DataError("ngram logprob: word id out of range")
        clen = min(len(context), self._order - 1)
        h = tuple(int(x) for x in context[len(context) - clen:]) if clen else ()
        bow10 = 0.0
        use = clen
        while True:
            e = self.find(h[len(h) - use:] + (word,))
            if e is not None:
                return (e[0] + bow10) * _LN10
            if use == 0:
                raise DataError("ngram logprob: missing unigram entry")
            c = self.find(h[len(h) - use:])
            if c is not None and c[2]:
                bow10 += c[1]
            use -= 1

    def prob(self, context, word) -> float:
        return math.exp(self.logprob(context, word))

    def shortlist(self, context: Sequence[int], k: int) -> List[int]:
        """The k most probable words, ties to the smaller id (ngram.hpp:213-252)."""
        if k < 1:
            raise ValueError("shortlist: k must be >= 1")
        if not self._unigram_desc:
            raise DataError("shortlist: model not finalized")
        clen = min(len(context), self._order - 1)
        h = tuple(int(x) for x in context[len(context) - clen:]) if clen else ()
        cands = set()
        for use in range(clen, 0, -1):
            cands.update(self._succ[use - 1].get(h[len(h) - use:], ()))
        cands = sorted(cands)
        pool = list(cands)
        taken = 0
        for w in self._unigram_desc:
            if taken >= k:
                break
            i = bisect_left(cands, w)
            if not (i < len(cands) and cands[i] == w):
                pool.append(w)
                taken += 1
        scored = sorted((-self.logprob(h, w), w) for w in pool)
        return [w for _, w in scored[:min(k, len(scored))]]


def estimate_kn(raw: List[Dict[tuple, int]], vocab_size: int, bos_id: int = 1) -> NGramModel:
    """Interpolated modified Kneser-Ney (ngram.hpp:336-426)."""
    order = len(raw)
    if order < 1:
        raise ValueError("estimate_kn: empty count table")
    if not raw[0]:
        raise DataError("estimate_kn: no unigram counts")
    V = vocab_size
    v_pred = V - 1
    model = NGramModel(order, V, bos_id)
    adj = adjust_counts(raw, bos_id)
    disc = [Discounts()] * (order + 1)
    for k in range(1, order + 1):
        n = [0] * 5
        for key, c in adj[k - 1].items():
            if k == 1 and key[0] == bos_id:
                continue
            if 1 <= c <= 4:
                n[c] += 1
        disc[k] = estimate_discounts(n)
    # unigram level
    a = [0] * V
    total = discounted = 0.0
    for key, c in adj[0].items():
        w = key[0]
        if w == bos_id:
            continue
        a[w] = c
        total += float(c)
        discounted += disc[1].of(c)
    if total <= 0.0:
        raise DataError("estimate_kn: no predictable unigrams")
    gamma = discounted / total
    p_uni = [0.0] * V
    for w in range(V):
        if w == bos_id:
            continue
        p_uni[w] = max(float(a[w]) - disc[1].of(a[w]), 0.0) / total + gamma / float(v_pred)
    lv0 = model.levels[0]
    for w in range(V):
        lv0[(w,)] = [LOG10_BOS_PROB if w == bos_id else math.log10(p_uni[w]), 0.0, False]
    p_low: Dict[tuple, float] = {(w,): p_uni[w] for w in range(V)}
    for k in range(2, order + 1):
        ctx: Dict[tuple, List[float]] = {}
        for key, c in adj[k - 1].items():
            st = ctx.setdefault(key[:-1], [0.0, 0.0])
            st[0] += float(c)
            st[1] += disc[k].of(c)
        lv = model.levels[k - 1]
        p_this: Dict[tuple, float] = {}
        for key, c in adj[k - 1].items():
            tot, dsc = ctx[key[:-1]]
            g = dsc / tot
            p = max(float(c) - disc[k].of(c), 0.0) / tot + g * p_low[key[1:]]
            p_this[key] = p
            lv[key] = [math.log10(p), 0.0, False]
        for hctx, (tot, dsc) in ctx.items():
            e = model.levels[k - 2][hctx]
            e[1] = math.log10(dsc / tot)
            e[2] = True
        p_low = p_this
    model.finalize()
    return model


def ngram_perplexity_full(model: NGramModel, ids: Sequence[int]):
    """stream_perplexity (ngram.hpp:430-451): context reset at bos, bos never
    predicted -> (total ln p, predicted, perplexity)."""
    total, pred, ctx = 0.0, 0, []
    maxc = model.order() - 1
    for w in ids:
        w = int(w)
        if w == model.bos_id:
            ctx = [w]
            continue
        total += model.logprob(ctx, w)
        pred += 1
        ctx.append(w)
        if maxc >= 0 and len(ctx) > maxc:
            ctx = ctx[len(ctx) - maxc:] if maxc > 0 else []
    if pred == 0:
        raise ValueError("perplexity: no predicted tokens")
    return total, pred, math.exp(-total / pred)
