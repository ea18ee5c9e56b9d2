"""Bottleneck / tied-embedding model (compress.hpp:38-415) on the device.

==============================  =============================================
this module                     reference (include/desklm/compress.hpp)
==============================  =============================================
``bottleneck_param_count``      ``bottleneck_param_count`` (:47-52)
``bn_init_uniform``             ``BottleneckParams::init_uniform`` (:78-82)
``GpuBottleneck``               ``BottleneckParams<float>`` +
                                ``BottleneckAdapter`` + ``BottleneckOptState``
``bn_bptt_run``                 ``bptt_run(BottleneckAdapter)``, softmax mode
                                (backprop.hpp:76-222)
``bottleneck_update``           ``bottleneck_update`` (:296-309)
``bn_sharded_perplexity``       ``sharded_perplexity(BottleneckAdapter)``
                                (eval.hpp:151-222)
``formats.write_bottleneck``    RNBL / RBOP byte layouts (:313-386)
==============================  =============================================

Every number comes from libdesklm_cuda.so (csrc/bottleneck.cu); this module
only moves host arrays across the C ABI (include/desklm_cuda.h, dl_bn_*).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import DL_BF16, DL_FP32, check, load

_PREC = {"fp32": DL_FP32, "bf16": DL_BF16}


def bottleneck_param_count(v: int, h: int, p: int) -> int:
    """compress.hpp:47-52: V*P + P*H + H*H + H*P."""
    if v < 1 or h < 1 or p < 1:
        raise ValueError("bottleneck param count: V,H,P >= 1")
    return v * p + p * h + h * h + h * p


def bn_init_uniform(V: int, H: int, P: int, seed: int, init_range: float = 0.1):
    """BottleneckParams::init_uniform (compress.hpp:78-82): one
    std::mt19937_64(seed) over e, u, w_rec, d in order (host, bit-exact)."""
    if V < 1 or H < 1 or P < 1:
        raise ValueError("BottleneckParams: V,H,P >= 1")
    if P > H:
        raise ValueError("BottleneckParams: P must not exceed H")
    from . import init_uniform  # the engine's host mt19937_64 stream
    # one generator over V*P + P*H + H*H + H*P values: the first n values of
    # the (n x 1) standard stream (its w_in) are exactly that sequence
    n = V * P + P * H + H * H + H * P
    flat = init_uniform(n, 1, seed, init_range)[0].ravel()
    sizes = [V * P, P * H, H * H, H * P]
    shapes = [(V, P), (P, H), (H, H), (H, P)]
    out, o = [], 0
    for sz, sh in zip(sizes, shapes):
        out.append(flat[o:o + sz].reshape(sh).copy())
        o += sz
    return tuple(out)


class _Res:
    def __init__(self, loss, positions):
        self.loss, self.positions = loss, positions


class GpuBottleneck:
    """Device-resident bottleneck model {E [V x P], U [P x H], W_rec [H x H],
    D [H x P]} with its rmsprop state.  precision: "fp32" (parity mode) or
    "bf16" (tcgen05 tensor cores; V, H, P multiples of 8)."""

    def __init__(self, V: int, H: int, P: int, act: int = 0, precision: str = "fp32",
                 device: int = 0):
        lib = load()
        self.V, self.H, self.P, self.act, self.precision = int(V), int(H), int(P), int(act), precision
        h = C.c_void_p()
        rc = lib.dl_bn_create(C.byref(h), device, self.V, self.H, self.P, self.act,
                              _PREC[precision])
        if rc:
            check_bn(rc, None)
        self._h = h
        self.rho, self.eps = 0.9995, 1e-6

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            load().dl_bn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        check_bn(rc, self._h)

    def _shapes(self):
        return ((self.V, self.P), (self.P, self.H), (self.H, self.H), (self.H, self.P))

    def set_params(self, e, u, w_rec, d):
        a = [np.ascontiguousarray(x, np.float32) for x in (e, u, w_rec, d)]
        if tuple(x.shape for x in a) != self._shapes():
            raise ValueError("set_params: shape mismatch")
        self._chk(load().dl_bn_set_params(self._h, *(x.ctypes.data for x in a)))

    def set_params_quantized(self, q):
        """RNQZ load (read_quantized + dequantize_model, compress.hpp:481-617):
        q is a formats.QuantizedModel; the codes are dequantised on the device."""
        if (q.v, q.h, q.p) != (self.V, self.H, self.P):
            raise ValueError("set_params_quantized: shape mismatch")

        class QM(C.Structure):
            _fields_ = [("bits", C.c_int), ("min", C.c_float), ("max", C.c_float),
                        ("codes", C.c_void_p)]

        bufs = [np.frombuffer(m.codes, np.uint8) for m in q.mats]
        arr = (QM * 4)(*[QM(m.bits, m.min, m.max, b.ctypes.data) for m, b in zip(q.mats, bufs)])
        self._chk(load().dl_bn_set_params_quantized(self._h, C.cast(arr, C.c_void_p)))

    def params(self):
        out = [np.empty(s, np.float32) for s in self._shapes()]
        self._chk(load().dl_bn_get_params(self._h, *(x.ctypes.data for x in out)))
        return tuple(out)

    def set_opt(self, m_e=None, m_u=None, m_rec=None, m_d=None, rho=0.9995, eps=1e-6):
        a = [None if x is None else np.ascontiguousarray(x, np.float32)
             for x in (m_e, m_u, m_rec, m_d)]
        self._chk(load().dl_bn_set_opt(self._h, *(None if x is None else x.ctypes.data
                                                  for x in a), rho, eps))
        self.rho, self.eps = rho, eps

    def opt(self):
        out = [np.empty(s, np.float32) for s in ((self.V,),) + self._shapes()[1:]]
        self._chk(load().dl_bn_get_opt(self._h, *(x.ctypes.data for x in out)))
        return tuple(out)

    def grads(self):
        """Clipped gradients of the last window: (g_e dense, g_u, g_rec, g_d)."""
        out = [np.empty(s, np.float32) for s in self._shapes()]
        self._chk(load().dl_bn_get_grads(self._h, *(x.ctypes.data for x in out)))
        return tuple(out)

    def launch_count(self) -> int:
        return int(load().dl_bn_launch_count(self._h))

    # ---- device-resident epoch schedule (dl_bn_trainer_*)
    def trainer_init(self, ids, noffset, minibatch, unroll, clip, bos=1):
        ids = np.ascontiguousarray(ids, np.uint32)
        self._chk(load().dl_bn_trainer_init(self._h, ids.ctypes.data, len(ids), noffset,
                                            minibatch, unroll, float(clip), bos))
        self._n_streams = noffset * minibatch

    def trainer_run(self, first, count, eta):
        """Windows [first, first+count) -> (loss sum, target positions, skipped)."""
        ls, pos, sk = C.c_double(0.0), C.c_uint64(0), C.c_uint64(0)
        self._chk(load().dl_bn_trainer_run(self._h, first, count, eta, C.byref(ls),
                                           C.byref(pos), C.byref(sk)))
        return ls.value, pos.value, sk.value

    def trainer_state(self):
        cur = np.empty(self._n_streams, np.int64)
        hid = np.empty((self._n_streams, self.H), np.float32)
        self._chk(load().dl_bn_trainer_get_state(self._h, cur.ctypes.data, hid.ctypes.data))
        return cur, hid

    def trainer_set_state(self, cursors, hidden):
        cur = np.ascontiguousarray(cursors, np.int64)
        hid = np.ascontiguousarray(hidden, np.float32)
        self._chk(load().dl_bn_trainer_set_state(self._h, cur.ctypes.data, hid.ctypes.data))

    # ---- NCE mode (the reference Trainer's default loss)
    def set_loss_mode(self, mode: int):
        """0 = NCE (LossMode::kNce), 1 = exact softmax."""
        self._chk(load().dl_bn_set_loss_mode(self._h, int(mode)))

    def set_noise(self, counts, k: int, floor: float = 1e-8):
        """NoiseModel over the vocabulary (nce.hpp:41-66) + AliasSampler."""
        c = np.ascontiguousarray(counts, np.float64)
        self._chk(load().dl_bn_set_noise(self._h, c.ctypes.data, len(c), int(k), float(floor)))

    def set_rng_state(self, state):
        st = np.ascontiguousarray(state, np.uint64)
        self._chk(load().dl_bn_set_rng_state(self._h, st.ctypes.data))

    def rng_state(self):
        st = np.zeros(313, np.uint64)
        self._chk(load().dl_bn_get_rng_state(self._h, st.ctypes.data))
        return st


def check_bn(rc, h):
    if rc == 0:
        return
    from ._lib import DL_EDATA, DL_EINVAL, DataError, DeviceError
    msg = (load().dl_bn_last_error(h) or b"").decode()
    if rc == DL_EINVAL:
        raise ValueError(msg)
    if rc == DL_EDATA:
        raise DataError(msg)
    raise DeviceError(msg)


def _window_arrays(model, wb, h0):
    x = np.ascontiguousarray(wb.inputs, np.uint32)
    y = np.ascontiguousarray(wb.targets, np.uint32)
    w = np.ascontiguousarray(wb.weights, np.uint8)
    if x.shape != y.shape or x.shape != w.shape or x.ndim != 2:
        raise ValueError("bptt: window size mismatch")
    T, B = x.shape
    h0 = np.ascontiguousarray(h0, np.float32)
    if h0.shape != (B, model.H):
        raise ValueError("bptt: initial state shape mismatch")
    return x, y, w, T, B, h0


def bn_bptt_run(model: GpuBottleneck, wb, h0, loss_scale: float = 1.0, clip: float = 1.0,
                compute_grads: bool = True):
    """bptt_run over the bottleneck adapter (softmax mode); returns
    (BpttResult, h_final); gradients stay on the device."""
    from . import BpttResult
    x, y, w, T, B, h0 = _window_arrays(model, wb, h0)
    hf = np.empty((B, model.H), np.float32)
    loss, pos = C.c_double(), C.c_uint64()
    model._chk(load().dl_bn_window(model.handle, T, B, x.ctypes.data, y.ctypes.data,
                                   w.ctypes.data, h0.ctypes.data, hf.ctypes.data,
                                   float(loss_scale), float(clip), int(compute_grads),
                                   C.byref(loss), C.byref(pos)))
    return BpttResult(loss.value, pos.value), hf


def bn_train_window(model: GpuBottleneck, wb, h0, loss_scale: float, clip: float, eta: float):
    """bptt_run + bottleneck_update in one call; (BpttResult, h_final, applied)."""
    from . import BpttResult
    x, y, w, T, B, h0 = _window_arrays(model, wb, h0)
    hf = np.empty((B, model.H), np.float32)
    loss, pos, applied = C.c_double(), C.c_uint64(), C.c_int()
    model._chk(load().dl_bn_train_window(model.handle, T, B, x.ctypes.data, y.ctypes.data,
                                         w.ctypes.data, h0.ctypes.data, hf.ctypes.data,
                                         float(loss_scale), float(clip), float(eta),
                                         C.byref(loss), C.byref(pos), C.byref(applied)))
    return BpttResult(loss.value, pos.value), hf, bool(applied.value)


def bottleneck_update(model: GpuBottleneck, eta: float) -> bool:
    applied = C.c_int()
    model._chk(load().dl_bn_rmsprop(model.handle, float(eta), C.byref(applied)))
    return bool(applied.value)


def bn_sharded_perplexity(model: GpuBottleneck, ids, shards: int, bos_id: int = 1):
    from . import PerplexityResult
    ids = np.ascontiguousarray(ids, np.uint32)
    tot, pred, ppl = C.c_double(), C.c_uint64(), C.c_double()
    model._chk(load().dl_bn_sharded_perplexity(model.handle, ids.ctypes.data, len(ids), shards,
                                               bos_id, C.byref(tot), C.byref(pred),
                                               C.byref(ppl)))
    return PerplexityResult(ppl.value, tot.value, pred.value)


class BottleneckTrainer:
    """Trainer<BottleneckTraits> (trainer.hpp:171-476 over compress.hpp:389-415),
    softmax (mode 1) or NCE (mode 0, the reference default).  The host keeps the reference's schedule -- offset-stream
    cursors floor(i*L/N), window (r, g) positions cursor + t, bos-masked
    targets, hidden carry and wrap reset (trainer.hpp:350-410).  By default
    the schedule itself is device resident (dl_bn_trainer_run: the epoch's
    windows are built, trained and carried on the device, softmax windows
    replayed from one CUDA graph); device_loop=False keeps it on the host
    and runs every window as one dl_bn_train_window call (bptt_run +
    bottleneck_update).  Validation is the device sharded scorer; the RTRN
    checkpoint carries RNBL + RBOP like the reference traits."""

    def __init__(self, cfg, params, vocab_words, train_ids, valid_ids, precision: str = "fp32",
                 device: int = 0, device_loop: bool = True):
        from . import BOS_ID, EpochLog  # noqa: F401
        cfg.validate()
        self.cfg = cfg
        self.vocab = list(vocab_words)
        e, u, w_rec, d = (np.asarray(x, np.float32) for x in params)
        V, P = e.shape
        H = w_rec.shape[0]
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
        L = len(self.train_ids)
        N = cfg.noffset * cfg.minibatch
        if L < N:
            raise ValueError("trainer: training stream shorter than the stream count")
        self.model = GpuBottleneck(V, H, P, cfg.act, precision, device)
        self.model.set_params(e, u, w_rec, d)
        self.model.set_opt(None, None, None, None, cfg.rho, cfg.eps)
        if cfg.mode == 0:
            # NoiseModel::from_stream over the non-bos training tokens and the
            # trainer's rng seeded with cfg.seed (trainer.hpp:184, 207-209)
            from . import rng_seed_state
            ids = self.train_ids
            counts = np.bincount(ids[ids != 1], minlength=V).astype(np.float64)
            self.model.set_loss_mode(0)
            self.model.set_noise(counts, cfg.nce_k, cfg.noise_floor)
            self.model.set_rng_state(rng_seed_state(cfg.seed))
        self.a0 = np.float32(0.5 if cfg.act == 0 else 0.0)
        self.device_loop = device_loop
        if device_loop:
            self.model.trainer_init(self.train_ids, cfg.noffset, cfg.minibatch, cfg.unroll,
                                    cfg.clip)
        else:
            self._cursors = np.array([i * L // N for i in range(N)], np.int64)
            self._hidden = np.full((N, H), self.a0, np.float32)
        self.logs = []
        self.epoch = 0
        self.bad_epochs = 0
        self.eta = cfg.eta
        self.best_ppl = 0.0
        self.initial_ppl = 0.0

    def params(self):
        return self.model.params()

    def validate(self) -> float:
        return bn_sharded_perplexity(self.model, self.valid, self.cfg.valid_shards).perplexity

    # the schedule's state (cursors, hidden carry): device resident unless
    # device_loop=False
    @property
    def cursors(self):
        return self.model.trainer_state()[0] if self.device_loop else self._cursors

    @property
    def hidden(self):
        return self.model.trainer_state()[1] if self.device_loop else self._hidden

    def _set_schedule(self, cursors, hidden):
        if self.device_loop:
            self.model.trainer_set_state(cursors, hidden)
        else:
            self._cursors = np.array(cursors, np.int64)
            self._hidden = np.array(hidden, np.float32)

    def run_epoch(self):
        """trainer.hpp:350-410 -> (mean window loss, skipped, tokens)."""
        cfg = self.cfg
        L = len(self.train_ids)
        B, T = cfg.minibatch, cfg.unroll
        N = cfg.noffset * B
        rounds = (L + N * T - 1) // (N * T)
        if self.device_loop:
            windows = rounds * cfg.noffset
            loss_sum, _, skipped = self.model.trainer_run(0, windows, self.eta)
            return (loss_sum / windows if windows else 0.0), skipped, rounds * N * T
        return self._run_epoch_host(rounds)

    def _run_epoch_host(self, rounds):
        from . import WindowBatch
        cfg = self.cfg
        ids, L = self.train_ids, len(self.train_ids)
        B, T = cfg.minibatch, cfg.unroll
        N = cfg.noffset * B
        tt = np.arange(T)[:, None]
        loss_sum, windows, skipped = 0.0, 0, 0
        for _ in range(rounds):
            for g in range(cfg.noffset):
                s0 = g * B
                pos = self._cursors[None, s0:s0 + B] + tt
                x = ids[pos % L]
                y = ids[(pos + 1) % L]
                w = (y != 1).astype(np.uint8)
                res, hf, ok = bn_train_window(self.model, WindowBatch(x, y, w),
                                              self._hidden[s0:s0 + B], 1.0 / (B * T), cfg.clip,
                                              self.eta)
                loss_sum += res.loss
                windows += 1
                skipped += 0 if ok else 1
                self._hidden[s0:s0 + B] = hf
                cur = self._cursors[s0:s0 + B]
                cur += T
                wrap = cur >= L
                cur[wrap] -= L
                self._hidden[s0:s0 + B][wrap] = self.a0
        return (loss_sum / windows if windows else 0.0), skipped, rounds * N * T

    def train(self, progress=None):
        """trainer.hpp:233-270 (the same loop as Trainer.train)."""
        from . import Trainer
        Trainer.train(self, progress)

    # ---- checkpointing (RTRN with RNBL / RBOP)
    def save_checkpoint(self) -> bytes:
        from . import formats
        rng_text = " ".join(str(int(v)) for v in self.model.rng_state()) \
            if self.cfg.mode == 0 else formats.mt19937_64_text(self.cfg.seed)
        return formats.write_trainer(self.cfg, self.epoch, self.eta, self.best_ppl,
                                     self.bad_epochs, self.initial_ppl, rng_text, self.cursors,
                                     self.hidden, self.model.params(), self.vocab,
                                     self.model.opt(), model="bottleneck")

    def load_checkpoint(self, data: bytes):
        from . import DataError, formats
        cfg = self.cfg
        st = formats.read_trainer(data, cfg, len(self.cursors), self.model.H,
                                  len(self.train_ids), model="bottleneck")
        e = st["params"][0]
        if st["params"][2].shape != (self.model.H, self.model.H) or e.shape[0] != self.model.V:
            raise DataError("trainer checkpoint: model shape mismatch")
        if st["vocab"] != self.vocab:
            raise DataError("trainer checkpoint: vocabulary mismatch")
        self.epoch, self.eta, self.best_ppl = st["epoch"], st["eta"], st["best"]
        self.bad_epochs, self.initial_ppl = st["bad"], st["initial"]
        self.model.set_params(*st["params"])
        self.model.set_opt(*st["opt"], cfg.rho, cfg.eps)
        self._set_schedule(st["cursors"], st["hidden"])
        if cfg.mode == 0:
            words = st["rng_text"].split()
            if len(words) != 313:
                raise DataError("trainer checkpoint: bad rng state")
            self.model.set_rng_state(np.array([int(v) for v in words], np.uint64))
