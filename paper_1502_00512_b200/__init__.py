"""desklm-b200: B200-native RNNLM trainer/scorer behind the desklm API.

Python mirror of the reference's public C++ interface for the training and
scoring path (paths relative to /root/reference/proj/include/desklm):

==========================  ===============================================
this package                reference
==========================  ===============================================
``GpuRnn``                  ``RnnParams<float>`` + ``StandardAdapter``
                            (rnn.hpp:61-84, :179-259), device-resident
``WindowBatch``             ``WindowBatch`` (backprop.hpp:36-50)
``bptt_run``                ``bptt_run`` softmax mode (backprop.hpp:76-222)
``rmsprop_update``          ``rmsprop_update`` (rmsprop.hpp:113-133)
``sharded_perplexity``      ``sharded_perplexity`` (eval.hpp:151-222)
``rnn_perplexity``          ``rnn_perplexity`` (eval.hpp:84-145)
``rescore_nbest``           ``rescore_nbest`` RNN part (eval.hpp:693-790)
``ln_z_samples``            ``ln_z_samples`` / ``drift_stats`` (eval.hpp:805-880)
``TrainConfig``/``Trainer`` ``TrainConfig``/``Trainer<StandardTraits>``
                            (trainer.hpp:43-93, :171-476)
``formats``                 RNLM / ROPT / RTRN (+ RNBL / RBOP) byte layouts
``bottleneck``              ``BottleneckParams`` / ``BottleneckAdapter`` /
                            ``bottleneck_update`` (compress.hpp:38-415)
==========================  ===============================================

Every number is computed by libdesklm_cuda.so (sm_100a kernels); this
module only moves host arrays across the C ABI.  Errors follow the
reference: ``ValueError`` for std::invalid_argument, ``DataError`` for
desklm::DataError.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import formats
from ._lib import DL_BF16, DL_FP32, DL_TF32X3, DataError, DeviceError, check, load

__all__ = [
    "GpuRnn", "WindowBatch", "BpttResult", "PerplexityResult", "bptt_run",
    "rmsprop_update", "train_window", "sharded_perplexity", "rng_seed_state", "rnn_perplexity", "score",
    "TrainConfig", "EpochLog", "Trainer", "DataError", "DeviceError", "formats",
    "param_count", "make_vocab", "KSIGMOID", "KTANH", "rescore_nbest",
    "read_nbest", "write_nbest", "NBestHyp", "NBestUtt", "ln_z_samples", "drift_stats",
    "DriftStats",
]

KSIGMOID, KTANH = 0, 1
UNK_ID, BOS_ID, EOS_ID = 0, 1, 2
_PREC = {"fp32": DL_FP32, "bf16": DL_BF16, "tf32x3": DL_TF32X3}


def _p(a):
    return None if a is None else a.ctypes.data


def param_count(v: int, h: int) -> int:
    """rnn.hpp:52-55: 2*V*H + H*H."""
    if v < 1 or h < 1:
        raise ValueError("param_count: V,H >= 1")
    return 2 * v * h + h * h


def make_vocab(v: int) -> List[str]:
    """Specials then w3, w4, ... (tests/oracles/helpers.hpp:26-31)."""
    return ["<unk>", "<s>", "</s>"] + [f"w{i}" for i in range(3, v)]


class GpuRnn:
    """Device-resident bias-free Elman RNNLM (V x H W_in, H x H W_rec, V x H
    word-major W_out) with its rmsprop state.  precision: "fp32" (parity
    mode, SIMT fp32 GEMMs), "tf32x3" (the fp32 mode with 3xTF32 tensor-core
    GEMMs) or "bf16" (tcgen05 tensor cores, bf16 operands)."""

    def __init__(self, V: int, H: int, act: int = KSIGMOID, precision: str = "fp32",
                 device: int = 0):
        lib = load()
        self.V, self.H, self.act, self.precision = int(V), int(H), int(act), precision
        h = C.c_void_p()
        check(lib.dl_create(C.byref(h), device, self.V, self.H, self.act, _PREC[precision]))
        self._h = h
        self.rho, self.eps = 0.9995, 1e-6

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            load().dl_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        check(rc, self._h)

    # ---- state
    def set_params(self, w_in, w_rec, w_out):
        a = [np.ascontiguousarray(x, np.float32) for x in (w_in, w_rec, w_out)]
        if a[0].shape != (self.V, self.H) or a[1].shape != (self.H, self.H) or \
                a[2].shape != (self.V, self.H):
            raise ValueError("set_params: shape mismatch")
        self._chk(load().dl_set_params(self._h, *(x.ctypes.data for x in a)))

    def params(self):
        w_in = np.empty((self.V, self.H), np.float32)
        w_rec = np.empty((self.H, self.H), np.float32)
        w_out = np.zeros((self.V, self.H), np.float32)  # vocab-sharded: own rows only
        self._chk(load().dl_get_params(self._h, w_in.ctypes.data, w_rec.ctypes.data,
                                       w_out.ctypes.data))
        return w_in, w_rec, w_out

    def set_opt(self, m_rec=None, m_in=None, m_out=None, rho=0.9995, eps=1e-6):
        a = [None if x is None else np.ascontiguousarray(x, np.float32)
             for x in (m_rec, m_in, m_out)]
        self._chk(load().dl_set_opt(self._h, *(_p(x) for x in a), rho, eps))
        self.rho, self.eps = rho, eps

    def opt(self):
        m_rec = np.empty((self.H, self.H), np.float32)
        m_in = np.empty(self.V, np.float32)
        m_out = np.zeros(self.V, np.float32)
        self._chk(load().dl_get_opt(self._h, m_rec.ctypes.data, m_in.ctypes.data,
                                    m_out.ctypes.data))
        return m_rec, m_in, m_out

    def grads(self):
        """Dense clipped gradients of the last window: (g_in, g_rec, g_out)."""
        g_in = np.empty((self.V, self.H), np.float32)
        g_rec = np.empty((self.H, self.H), np.float32)
        g_out = np.zeros((self.V, self.H), np.float32)
        self._chk(load().dl_get_grads(self._h, g_in.ctypes.data, g_rec.ctypes.data,
                                      g_out.ctypes.data))
        return g_in, g_rec, g_out

    def set_grads(self, in_words, in_rows, g_rec, g_out):
        """Test hook: StandardGrads (sparse W_in rows, dense W_rec/W_out)."""
        w = np.ascontiguousarray(in_words, np.uint32)
        r = np.ascontiguousarray(in_rows, np.float32).reshape(len(w), self.H)
        gr = np.ascontiguousarray(g_rec, np.float32)
        go = np.ascontiguousarray(g_out, np.float32)
        self._chk(load().dl_set_grads(self._h, len(w), w.ctypes.data, r.ctypes.data,
                                      gr.ctypes.data, go.ctypes.data))

    def launch_count(self) -> int:
        return int(load().dl_launch_count(self._h))

    def set_profiling(self, on: bool):
        self._chk(load().dl_set_profiling(self._h, int(on)))

    def kernel_ms(self, name: str) -> float:
        return float(load().dl_kernel_ms(self._h, name.encode()))

    # ---- trainer plumbing
    def trainer_init(self, ids, noffset, minibatch, unroll, clip, bos=BOS_ID):
        ids = np.ascontiguousarray(ids, np.uint32)
        self._chk(load().dl_trainer_init(self._h, ids.ctypes.data, len(ids), noffset,
                                         minibatch, unroll, float(clip), bos))
        self._n_local = noffset * minibatch

    def trainer_run(self, first, count, eta):
        ls, sk = C.c_double(0.0), C.c_uint64(0)
        self._chk(load().dl_trainer_run(self._h, first, count, eta, C.byref(ls), C.byref(sk)))
        return ls.value, sk.value

    def trainer_state(self):
        cur = np.empty(self._n_local, np.int64)
        hid = np.empty((self._n_local, self.H), np.float32)
        self._chk(load().dl_trainer_get_state(self._h, cur.ctypes.data, hid.ctypes.data))
        return cur, hid

    def trainer_set_state(self, cursors, hidden):
        cur = np.ascontiguousarray(cursors, np.int64)
        hid = np.ascontiguousarray(hidden, np.float32)
        self._chk(load().dl_trainer_set_state(self._h, cur.ctypes.data, hid.ctypes.data))

    def comm_init_local(self, group: "LocalGroup", rank: int):
        """Join an in-process rank group (single-device multi-rank runs)."""
        self._chk(load().dl_comm_init_local(self._h, group.handle, rank))
        self._group = group  # keep the group alive as long as the model

    def comm_init(self, unique_id: bytes, nranks: int, rank: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        self._chk(load().dl_comm_init(self._h, C.addressof(buf), nranks, rank))

    def set_loss_mode(self, mode: int):
        """0 = NCE (LossMode::kNce), 1 = exact softmax (dl_set_loss_mode)."""
        self._chk(load().dl_set_loss_mode(self._h, int(mode)))

    def set_noise(self, counts, k: int, floor: float = 1e-8):
        """NoiseModel(counts, k, floor) (nce.hpp:41-66) for NCE windows."""
        c = np.ascontiguousarray(counts, np.float64)
        self._chk(load().dl_set_noise(self._h, c.ctypes.data, len(c), int(k), float(floor)))

    def set_rng_state(self, state):
        st = np.ascontiguousarray(state, np.uint64)
        if st.shape != (313,):
            raise ValueError("rng state: 313 uint64 (312 words + position)")
        self._chk(load().dl_set_rng_state(self._h, st.ctypes.data))

    def rng_state(self):
        st = np.zeros(313, np.uint64)
        self._chk(load().dl_get_rng_state(self._h, st.ctypes.data))
        return st

    def set_vocab_shard(self, on=True):
        """Vocabulary-sharded softmax over the communicator's ranks
        (dl_set_vocab_shard): this rank keeps W_out rows [r*V/G, (r+1)*V/G).
        on=True / 1: every rank runs the same streams; on="dp" / 2: data-
        parallel streams with a vocabulary-parallel output layer over the
        gathered window.  Zeroes W_out / m_out -- call before set_params."""
        mode = 2 if on == "dp" else int(on)
        self._chk(load().dl_set_vocab_shard(self._h, mode))


def rng_seed_state(seed: int):
    """std::mt19937_64(seed) as 312 state words + position (uint64[313])."""
    st = np.zeros(313, np.uint64)
    check(load().dl_rng_seed_state(int(seed), st.ctypes.data))
    return st


def init_uniform(V: int, H: int, seed: int, init_range: float = 0.1):
    """RnnParams<float>::init_uniform (rnn.hpp:79-83), bit-identical (host
    C-ABI call, std::mt19937_64).  Returns (w_in, w_rec, w_out)."""
    w_in = np.empty((V, H), np.float32)
    w_rec = np.empty((H, H), np.float32)
    w_out = np.empty((V, H), np.float32)
    check(load().dl_init_uniform(V, H, seed, init_range, w_in.ctypes.data, w_rec.ctypes.data,
                                 w_out.ctypes.data))
    return w_in, w_rec, w_out


def rank_cursors(L: int, noffset: int, minibatch: int, nranks: int = 1, rank: int = 0):
    """This rank's initial stream cursors (host-only C-ABI call): the
    reference's floor(i*L/N) (trainer.hpp:194-195) over global streams
    i = g*nranks*minibatch + rank*minibatch + b, group-major."""
    out = np.empty(noffset * minibatch, np.int64)
    check(load().dl_rank_cursors(L, noffset, minibatch, nranks, rank, out.ctypes.data))
    return out


class LocalGroup:
    """G contexts on one device acting as G ranks (dl_local_group_create);
    drive each rank's calls from its own thread (collectives synchronise the
    host threads)."""

    def __init__(self, G: int):
        h = C.c_void_p()
        check(load().dl_local_group_create(G, C.byref(h)))
        self.handle, self.G = h, G

    def __del__(self):
        try:
            if self.handle:
                load().dl_local_group_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def comm_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(load().dl_comm_unique_id(C.addressof(buf)))
    return bytes(buf)


@dataclass
class WindowBatch:
    """t-major window (index t*B+b); weights 0 mask a position out."""
    inputs: np.ndarray
    targets: np.ndarray
    weights: np.ndarray

    @property
    def T(self):
        return self.inputs.shape[0]

    @property
    def B(self):
        return self.inputs.shape[1]


@dataclass
class BpttResult:
    loss: float = 0.0
    positions: int = 0


@dataclass
class PerplexityResult:
    perplexity: float = 0.0
    total_logprob: float = 0.0
    predicted: int = 0


def bptt_run(model: GpuRnn, wb: WindowBatch, h0, loss_scale: float = 1.0,
             clip: float = 1.0, compute_grads: bool = True):
    """Softmax-mode bptt_run; returns (BpttResult, h_final).  Gradients stay
    on the device for rmsprop_update / GpuRnn.grads()."""
    x = np.ascontiguousarray(wb.inputs, np.uint32)
    y = np.ascontiguousarray(wb.targets, np.uint32)
    w = np.ascontiguousarray(wb.weights, np.uint8)
    if x.shape != y.shape or x.shape != w.shape or x.ndim != 2:
        raise ValueError("bptt: window size mismatch")
    T, B = x.shape
    h0 = np.ascontiguousarray(h0, np.float32)
    if h0.shape != (B, model.H):
        raise ValueError("bptt: initial state shape mismatch")
    hf = np.empty((B, model.H), np.float32)
    loss, pos = C.c_double(), C.c_uint64()
    model._chk(load().dl_window(model.handle, T, B, x.ctypes.data, y.ctypes.data,
                                w.ctypes.data, h0.ctypes.data, hf.ctypes.data,
                                float(loss_scale), float(clip), int(compute_grads),
                                C.byref(loss), C.byref(pos)))
    return BpttResult(loss.value, pos.value), hf


def train_window(model: GpuRnn, wb: WindowBatch, h0, loss_scale: float, clip: float,
                 eta: float, h_final=None):
    """One Trainer::run_epoch step (trainer.hpp:391-397): bptt_run then
    rmsprop_update in one call (dl_train_window); returns (BpttResult,
    h_final, applied).  h_final: optional float32 [B, H] output buffer
    (page-locked buffers -- inputs too -- are DMA'd without staging)."""
    x = np.ascontiguousarray(wb.inputs, np.uint32)
    y = np.ascontiguousarray(wb.targets, np.uint32)
    w = np.ascontiguousarray(wb.weights, np.uint8)
    if x.shape != y.shape or x.shape != w.shape or x.ndim != 2:
        raise ValueError("bptt: window size mismatch")
    T, B = x.shape
    h0 = np.ascontiguousarray(h0, np.float32)
    if h0.shape != (B, model.H):
        raise ValueError("bptt: initial state shape mismatch")
    hf = np.empty((B, model.H), np.float32) if h_final is None else h_final
    if hf.shape != (B, model.H) or hf.dtype != np.float32 or not hf.flags.c_contiguous:
        raise ValueError("h_final: float32 [B, H] C-contiguous buffer expected")
    loss, pos, applied = C.c_double(), C.c_uint64(), C.c_int()
    model._chk(load().dl_train_window(model.handle, T, B, x.ctypes.data, y.ctypes.data,
                                      w.ctypes.data, h0.ctypes.data, hf.ctypes.data,
                                      float(loss_scale), float(clip), float(eta),
                                      C.byref(loss), C.byref(pos), C.byref(applied)))
    return BpttResult(loss.value, pos.value), hf, bool(applied.value)


def rmsprop_update(model: GpuRnn, eta: float) -> bool:
    applied = C.c_int()
    model._chk(load().dl_rmsprop(model.handle, float(eta), C.byref(applied)))
    return bool(applied.value)


def score(model: GpuRnn, inputs, targets, h0=None):
    """Lock-step scorer: inputs/targets [steps x S] (targets -1 = skip).
    Returns (logp [steps x S] with NaN where skipped, total, predicted, h_final)."""
    x = np.ascontiguousarray(inputs, np.uint32)
    t = np.ascontiguousarray(targets, np.int64)
    steps, S = x.shape
    lp = np.empty((steps, S), np.float64)
    hf = np.empty((S, model.H), np.float32)
    tot, pred = C.c_double(), C.c_uint64()
    h0a = None if h0 is None else np.ascontiguousarray(h0, np.float32)
    model._chk(load().dl_score(model.handle, S, steps, x.ctypes.data, t.ctypes.data, _p(h0a),
                               hf.ctypes.data, lp.ctypes.data, C.byref(tot), C.byref(pred)))
    return lp, tot.value, pred.value, hf


def sharded_perplexity(model: GpuRnn, ids, shards: int, bos_id: int = BOS_ID):
    ids = np.ascontiguousarray(ids, np.uint32)
    tot, pred, ppl = C.c_double(), C.c_uint64(), C.c_double()
    model._chk(load().dl_sharded_perplexity(model.handle, ids.ctypes.data, len(ids), shards,
                                            bos_id, C.byref(tot), C.byref(pred), C.byref(ppl)))
    return PerplexityResult(ppl.value, tot.value, pred.value)


def ln_z_samples(model: GpuRnn, ids, count: int) -> np.ndarray:
    """ln_z_samples (eval.hpp:805-857): ln Z of up to `count` hidden states
    sampled at stride max(1, n / count) from one pass over the stream."""
    ids = np.ascontiguousarray(ids, np.uint32)
    out = np.empty(max(int(count), 1), np.float64)
    n = C.c_int64()
    model._chk(load().dl_ln_z_samples(model.handle, ids.ctypes.data, len(ids), int(count),
                                      out.ctypes.data, C.byref(n)))
    return out[: n.value].copy()


@dataclass
class DriftStats:
    mean: float = 0.0
    median: float = 0.0
    q25: float = 0.0
    q75: float = 0.0
    iqr: float = 0.0
    contexts: int = 0


def drift_stats(ln_z) -> DriftStats:
    """drift_stats (eval.hpp:859-880): mean and linearly interpolated
    quartiles of the sorted samples (host arithmetic, same order)."""
    v = sorted(float(x) for x in ln_z)
    if len(v) < 100:
        raise ValueError("drift stats: need at least 100 contexts")
    total = 0.0
    for x in v:
        total += x

    def quantile(q):
        pos = q * float(len(v) - 1)
        lo = int(pos)
        frac = pos - float(lo)
        if lo + 1 >= len(v):
            return v[-1]
        return v[lo] * (1.0 - frac) + v[lo + 1] * frac

    q25, q75 = quantile(0.25), quantile(0.75)
    return DriftStats(total / float(len(v)), quantile(0.5), q25, q75, q75 - q25, len(v))


def rnn_perplexity(model: GpuRnn, ids, bos_id: int = BOS_ID):
    ids = np.ascontiguousarray(ids, np.uint32)
    tot, pred, ppl = C.c_double(), C.c_uint64(), C.c_double()
    model._chk(load().dl_rnn_perplexity(model.handle, ids.ctypes.data, len(ids), bos_id,
                                        C.byref(tot), C.byref(pred), C.byref(ppl)))
    return PerplexityResult(ppl.value, tot.value, pred.value)


# ----------------------------------------------------------------- n-best
@dataclass
class NBestHyp:
    acoustic: float = 0.0
    old_lm: float = 0.0
    words: List[str] = field(default_factory=list)
    new_lm: float = 0.0
    new_total: float = 0.0
    rank: int = 0


@dataclass
class NBestUtt:
    id: str
    hyps: List[NBestHyp]


def read_nbest(text: str) -> List[NBestUtt]:
    """eval.hpp:612-657: `utt<TAB>acoustic<TAB>old-lm[<TAB>words]` (3, 4 or 7
    fields); consecutive lines with one id form an utterance."""
    utts: List[NBestUtt] = []
    for ln, line in enumerate(text.split("\n"), 1):
        if line.endswith("\r"):
            line = line[:-1]
        if not line:
            continue
        f = line.split("\t")
        if len(f) not in (3, 4, 7):
            raise DataError(f"expected 3, 4, or 7 tab-separated fields, got {len(f)} (line {ln})")
        if not f[0]:
            raise DataError(f"empty utterance id (line {ln})")
        try:
            h = NBestHyp(float(f[1]), float(f[2]))
        except ValueError:
            raise DataError(f"expected a number (line {ln})")
        if len(f) >= 4:
            h.words = [w for w in f[3].split(" ") if w]
        if not utts or utts[-1].id != f[0]:
            utts.append(NBestUtt(f[0], []))
        utts[-1].hyps.append(h)
    return utts


def write_nbest(utts: Sequence[NBestUtt]) -> str:
    """eval.hpp:660-677."""
    out = []
    for u in utts:
        for h in u.hyps:
            out.append(f"{u.id}\t{h.acoustic:.6f}\t{h.old_lm:.6f}\t{' '.join(h.words)}\t"
                       f"{h.new_lm:.6f}\t{h.new_total:.6f}\t{h.rank}\n")
    return "".join(out)


def rescore_nbest(utts: List[NBestUtt], model: GpuRnn, vocab_words: Sequence[str],
                  lm_scale: float = 1.0, wip: float = 0.0) -> None:
    """RNN-only exact rescoring (eval.hpp:693-790 with ngram == nullptr):
    every hypothesis is one stream (bos + words + eos, h = act(0)); all
    hypotheses are scored together by the lock-step device scorer."""
    index = {w: i for i, w in enumerate(vocab_words)}
    hyps = [h for u in utts for h in u.hyps]
    if not hyps:
        return
    seqs = [[BOS_ID] + [index.get(w, UNK_ID) for w in h.words] + [EOS_ID] for h in hyps]
    steps = max(len(s) for s in seqs) - 1
    S = len(seqs)
    x = np.zeros((steps, S), np.uint32)
    t = np.full((steps, S), -1, np.int64)
    for s, ids in enumerate(seqs):
        n = len(ids) - 1
        x[:n, s] = ids[:-1]
        t[:n, s] = ids[1:]
    lp, _, _, _ = score(model, x, t)
    for s, h in enumerate(hyps):
        n = len(seqs[s]) - 1
        total = 0.0
        for j in range(n):  # (j) order per hypothesis, as the reference sums
            total += float(lp[j, s])
        h.new_lm = total
        h.new_total = h.acoustic + lm_scale * total + wip * len(h.words)
    for u in utts:
        u.hyps.sort(key=lambda h: -h.new_total)  # stable, like std::stable_sort
        for i, h in enumerate(u.hyps):
            h.rank = i + 1


# ---------------------------------------------------------------- trainer
@dataclass
class TrainConfig:
    """trainer.hpp:43-93, same defaults.  mode: 0 = NCE (LossMode::kNce, the
    reference's default, trainer.hpp:53: k = nce_k noise samples per position
    from the unigram NoiseModel), 1 = exact softmax."""
    nstate: int = 256
    nproj: int = 0
    noffset: int = 128
    minibatch: int = 8
    unroll: int = 16
    eta: float = 1e-3
    rho: float = 0.9995
    eps: float = 1e-6
    clip: float = 1.0
    mode: int = 0
    nce_k: int = 64
    noise_floor: float = 1e-8
    max_epochs: int = 20
    seed: int = 1
    act: int = KSIGMOID
    divergence_factor: float = 10.0
    valid_limit: int = 0
    valid_shards: int = 8
    init_range: float = 0.1
    threads: int = 1

    def validate(self):
        if self.nstate < 1:
            raise ValueError("config: nstate must be >= 1")
        if self.nproj < 0:
            raise ValueError("config: nproj must be >= 0")
        if self.noffset < 1 or self.minibatch < 1 or self.unroll < 1:
            raise ValueError("config: noffset, minibatch, unroll must be >= 1")
        if not self.eta > 0.0:
            raise ValueError("config: eta must be > 0")
        if not (0.0 < self.rho < 1.0):
            raise ValueError("config: rho must be in (0, 1)")
        if not self.eps > 0.0:
            raise ValueError("config: eps must be > 0")
        if not self.clip > 0.0:
            raise ValueError("config: clip must be > 0")
        if self.mode == 0 and self.nce_k < 1:
            raise ValueError("config: nce_k must be >= 1")
        if not self.noise_floor > 0.0:
            raise ValueError("config: noise_floor must be > 0")
        if self.max_epochs < 1:
            raise ValueError("config: max_epochs must be >= 1")
        if not self.divergence_factor > 1.0:
            raise ValueError("config: divergence_factor must be > 1")
        if self.valid_limit < 0:
            raise ValueError("config: valid_limit must be >= 0")
        if self.valid_shards < 1:
            raise ValueError("config: valid_shards must be >= 1")
        if not self.init_range > 0.0:
            raise ValueError("config: init_range must be > 0")
        if self.threads < 1:
            raise ValueError("config: threads must be >= 1")
        if self.mode not in (0, 1):
            raise ValueError("config: mode must be 0 (NCE) or 1 (softmax)")


@dataclass
class EpochLog:
    epoch: int = 0
    train_loss: float = 0.0
    valid_ppl: float = 0.0
    eta: float = 0.0
    seconds: float = 0.0
    tokens_per_sec: float = 0.0
    skipped_updates: int = 0


def write_epoch_log(logs: Sequence[EpochLog]) -> str:
    """trainer.hpp:105-115."""
    out = ["epoch,train_loss,valid_ppl,eta,seconds,tokens_per_sec,skipped\n"]
    for l in logs:
        out.append("%d,%.6f,%.4f,%.8g,%.2f,%.1f,%d\n" % (
            l.epoch, l.train_loss, l.valid_ppl, l.eta, l.seconds, l.tokens_per_sec,
            l.skipped_updates))
    return "".join(out)


class Trainer:
    """Trainer<StandardTraits> (trainer.hpp:171-476) with the epoch loop on the
    device: offset-stream cursors, hidden carry, window build, bptt_run,
    rmsprop and wrap reset all run inside libdesklm_cuda (one CUDA graph per
    window).  Validation is the device sharded scorer."""

    def __init__(self, cfg: TrainConfig, params, vocab_words: Sequence[str], train_ids,
                 valid_ids, precision: str = "fp32", device: int = 0, comm=None,
                 vocab_shard=False):
        cfg.validate()
        self.cfg = cfg
        self.vocab = list(vocab_words)
        w_in, w_rec, w_out = params
        V, H = np.asarray(w_in).shape
        if len(self.vocab) != V:
            raise ValueError("trainer: vocabulary/model size mismatch")
        if H != cfg.nstate:
            raise ValueError("trainer: nstate does not match the parameters")
        self.train_ids = np.ascontiguousarray(train_ids, np.uint32)
        valid = np.ascontiguousarray(valid_ids, np.uint32)
        if cfg.valid_limit > 0 and len(valid) > cfg.valid_limit:
            valid = valid[: cfg.valid_limit]
        if len(valid) < 2:
            raise ValueError("trainer: validation stream too short")
        self.valid = valid
        self.nranks, self.rank = (1, 0) if comm is None else (comm[1], comm[2])
        # vocabulary-sharded ranks (vocab_shard=True) all run the same
        # streams; data-parallel ranks -- plain, or with the vocabulary-
        # parallel output layer (vocab_shard="dp") -- split the global minibatch
        self.dp_ranks = 1 if vocab_shard is True else self.nranks
        L = len(self.train_ids)
        N = cfg.noffset * cfg.minibatch * self.dp_ranks
        if L < N:
            raise ValueError("trainer: training stream shorter than the stream count")
        self.model = GpuRnn(V, H, cfg.act, precision, device)
        # comm: (nccl_unique_id, nranks, rank) or (LocalGroup, nranks, rank)
        if comm is not None and isinstance(comm[0], LocalGroup):
            self.model.comm_init_local(comm[0], comm[2])
        elif comm is not None:
            self.model.comm_init(comm[0], comm[1], comm[2])
        self.model_sharded = bool(vocab_shard)
        if vocab_shard:
            self.model.set_vocab_shard(vocab_shard)
        self.model.set_params(w_in, w_rec, w_out)
        self.model.set_opt(None, None, None, cfg.rho, cfg.eps)
        if cfg.mode == 0:
            # NoiseModel::from_stream (nce.hpp:69-76; trainer.hpp:207-209):
            # every non-bos token of the training stream; Trainer::rng_ is
            # seeded with cfg.seed (trainer.hpp:184)
            ids = self.train_ids
            counts = np.bincount(ids[ids != BOS_ID], minlength=V).astype(np.float64)
            self.model.set_loss_mode(0)
            self.model.set_noise(counts, cfg.nce_k, cfg.noise_floor)
            self.model.set_rng_state(rng_seed_state(cfg.seed))
        self.model.trainer_init(self.train_ids, cfg.noffset, cfg.minibatch, cfg.unroll,
                                cfg.clip)
        self.logs: List[EpochLog] = []
        self.epoch = 0
        self.bad_epochs = 0
        self.eta = cfg.eta
        self.best_ppl = 0.0
        self.initial_ppl = 0.0

    def params(self):
        return self.model.params()

    def validate(self) -> float:
        return sharded_perplexity(self.model, self.valid, self.cfg.valid_shards).perplexity

    def run_epoch(self):
        """trainer.hpp:350-410 -> (mean window loss, skipped, tokens)."""
        cfg = self.cfg
        L = len(self.train_ids)
        N = cfg.noffset * cfg.minibatch * self.dp_ranks
        T = cfg.unroll
        rounds = (L + N * T - 1) // (N * T)
        windows = rounds * cfg.noffset
        loss_sum, skipped = self.model.trainer_run(0, windows, self.eta)
        return (loss_sum / windows if windows > 0 else 0.0), skipped, rounds * N * T

    def train(self, progress=None):
        """trainer.hpp:233-270."""
        if self.initial_ppl == 0.0:
            self.initial_ppl = self.validate()
            self.best_ppl = self.initial_ppl
            if progress:
                progress(f"initial valid ppl {self.initial_ppl}")
        cfg = self.cfg
        while self.epoch < cfg.max_epochs and self.bad_epochs < 2:
            t0 = time.perf_counter()
            mean_loss, skipped, tokens = self.run_epoch()
            ppl = self.validate()
            secs = time.perf_counter() - t0
            self.epoch += 1
            log = EpochLog(self.epoch, mean_loss, ppl, self.eta, secs,
                           tokens / secs if secs > 0 else 0.0, skipped)
            self.logs.append(log)
            if progress:
                progress(f"epoch {log.epoch} loss {log.train_loss} valid ppl {ppl} eta {log.eta}")
            if ppl > cfg.divergence_factor * self.initial_ppl:
                raise DataError(f"trainer: diverged (validation perplexity {ppl} vs initial "
                                f"{self.initial_ppl})")
            if ppl < self.best_ppl:
                self.best_ppl = ppl
                self.bad_epochs = 0
            else:
                self.bad_epochs += 1
                self.eta *= 0.5

    # ---- checkpointing (RTRN, trainer.hpp:274-341)
    def _single_rank_only(self, what):
        # a rank holds only its own streams' cursors / hidden state (and, with
        # a vocabulary-sharded output layer, its own W_out / m_out rows): an
        # RTRN blob written by one rank is not the run's checkpoint
        if self.nranks > 1:
            raise NotImplementedError(
                f"{what}: RTRN checkpoints of multi-rank trainers are not supported "
                f"(each rank holds 1/{self.nranks} of the streams"
                + (" and of W_out" if self.model_sharded else "") + ")")

    def save_checkpoint(self) -> bytes:
        self._single_rank_only("save_checkpoint")
        cur, hid = self.model.trainer_state()
        # the rng as `os << rng_` (trainer.hpp:284): it only advances in NCE mode
        rng_text = " ".join(str(int(v)) for v in self.model.rng_state()) \
            if self.cfg.mode == 0 else formats.mt19937_64_text(self.cfg.seed)
        return formats.write_trainer(self.cfg, self.epoch, self.eta, self.best_ppl,
                                     self.bad_epochs, self.initial_ppl, rng_text, cur, hid,
                                     self.model.params(), self.vocab, self.model.opt())

    def load_checkpoint(self, data: bytes):
        self._single_rank_only("load_checkpoint")
        cfg = self.cfg
        n = cfg.noffset * cfg.minibatch
        st = formats.read_trainer(data, cfg, n, self.model.H, len(self.train_ids))
        w_in = st["params"][0]
        if w_in.shape != (self.model.V, self.model.H):
            raise DataError("trainer checkpoint: model shape mismatch")
        if st["vocab"] != self.vocab:
            raise DataError("trainer checkpoint: vocabulary mismatch")
        self.epoch, self.eta, self.best_ppl = st["epoch"], st["eta"], st["best"]
        self.bad_epochs, self.initial_ppl = st["bad"], st["initial"]
        self.model.set_params(*st["params"])
        self.model.set_opt(*st["opt"], cfg.rho, cfg.eps)
        self.model.trainer_set_state(st["cursors"], st["hidden"])
        if cfg.mode == 0:
            words = st["rng_text"].split()
            if len(words) != 313:
                raise DataError("trainer checkpoint: bad rng state")
            self.model.set_rng_state(np.array([int(v) for v in words], np.uint64))
