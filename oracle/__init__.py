"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the RNNLM hot path.

Two interchangeable back ends with one numpy-facing API:

* ``Orc``  -- ``oracle/liborc.so``: a plain-C restatement of the reference
  algorithm (``oracle/desklm_oracle.c``, every function cites the reference
  file:line it restates).
* ``Ref``  -- ``oracle/_ref/libdesklm_ref.so``: the unmodified reference
  headers (``/root/reference/proj/include``) compiled behind a C shim
  (``oracle/ref_shim.cpp``).  Built here; the prebuilt ``.so`` travels to
  the GPU box, where ``/root/reference`` itself does not exist.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package; the product library never calls it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(_HERE, "liborc.so")
REF_SO = os.path.join(_HERE, "_ref", "libdesklm_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_i64 = C.c_int64
_u64 = C.c_uint64


class TrainConfig(C.Structure):
    """Field order of the RTRN config echo (trainer.hpp:412-432); defaults
    follow TrainConfig (trainer.hpp:43-63), NCE mode included."""

    _fields_ = [
        ("nstate", C.c_int64), ("nproj", C.c_int64),
        ("noffset", C.c_int32), ("minibatch", C.c_int32),
        ("unroll", C.c_int32), ("mode", C.c_int32),
        ("eta", C.c_double), ("rho", C.c_double), ("eps", C.c_double),
        ("clip", C.c_double), ("nce_k", C.c_int32), ("max_epochs", C.c_int32),
        ("noise_floor", C.c_double), ("seed", C.c_uint64),
        ("act", C.c_int32), ("valid_shards", C.c_int32),
        ("divergence_factor", C.c_double), ("valid_limit", C.c_int64),
        ("init_range", C.c_double), ("threads", C.c_int32), ("pad_", C.c_int32),
    ]

    def __init__(self, **kw):
        d = dict(nstate=256, nproj=0, noffset=128, minibatch=8, unroll=16,
                 mode=0, eta=1e-3, rho=0.9995, eps=1e-6, clip=1.0, nce_k=64,
                 max_epochs=20, noise_floor=1e-8, seed=1, act=0,
                 valid_shards=8, divergence_factor=10.0, valid_limit=0,
                 init_range=0.1, threads=1, pad_=0)
        d.update(kw)
        super().__init__(**d)


def build(quiet: bool = True) -> None:
    """Compile liborc.so (and _ref when /root/reference is present)."""
    out = subprocess.run(["make", "-C", _HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


class _Backend:
    prefix = ""
    so_path = ""

    def __init__(self):
        if not os.path.exists(self.so_path):
            raise FileNotFoundError(f"{self.so_path} not built (make -C oracle)")
        self.lib = C.CDLL(self.so_path)
        p = self.prefix
        L = self.lib
        self._bptt = getattr(L, p + "bptt")
        self._bptt.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _i64, _i64,
                               _u32p, _u32p, _u8p, _f32p, C.c_double, C.c_float,
                               C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, _vp,
                               C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        self._rms = getattr(L, p + "rmsprop")
        self._rms.argtypes = [_i64, _i64, _f32p, _f32p, _f32p, _f32p, _f32p, _f32p,
                              C.c_double, C.c_double, C.c_double, _i64, _vp, _vp,
                              _f32p, C.c_int, _i64, _vp, _vp, C.POINTER(C.c_int)]
        self._init = getattr(L, p + "init_uniform")
        self._init.argtypes = [_i64, _i64, _u64, C.c_double, _f32p, _f32p, _f32p]
        self._rs = getattr(L, p + "random_stream")
        self._rs.restype = C.c_int64
        self._rs.argtypes = [_u64, _u64, _u64, _u64, _vp, _u64]
        self._rsp = getattr(L, p + "random_stream_pair")
        self._rsp.argtypes = [_u64, _u64, _u64, _u64, _vp, _u64, C.POINTER(C.c_int64),
                              _vp, _u64, C.POINTER(C.c_int64)]
        self._sppl = getattr(L, p + "sharded_ppl")
        self._sppl.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _u32p, _i64,
                               C.c_int, C.c_uint32, C.c_int, C.POINTER(C.c_double),
                               C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        self._rppl = getattr(L, p + "rnn_ppl")
        self._rppl.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _u32p, _i64,
                               C.c_uint32, C.c_int, C.POINTER(C.c_double),
                               C.POINTER(C.c_uint64), C.POINTER(C.c_double)]

    def _check(self, rc):
        if rc != 0:
            msg = ""
            if hasattr(self.lib, "ref_last_error"):
                self.lib.ref_last_error.restype = C.c_char_p
                msg = self.lib.ref_last_error().decode()
            raise OracleError(rc, msg)

    # ---- data helpers
    def init_uniform(self, V, H, seed, rng=0.1):
        w_in = np.empty((V, H), np.float32)
        w_rec = np.empty((H, H), np.float32)
        w_out = np.empty((V, H), np.float32)
        self._check(self._init(V, H, seed, rng, w_in, w_rec, w_out))
        return w_in, w_rec, w_out

    def random_stream(self, seed, v, min_tokens, max_len=12):
        n = self._rs(seed, v, min_tokens, max_len, None, 0)
        out = np.empty(n, np.uint32)
        self._rs(seed, v, min_tokens, max_len, out.ctypes.data, n)
        return out

    def random_stream_pair(self, seed, v, min_a, min_b):
        la, lb = C.c_int64(), C.c_int64()
        cap = 2 * (min_a + min_b) + 64
        a = np.empty(cap, np.uint32)
        b = np.empty(cap, np.uint32)
        self._check(self._rsp(seed, v, min_a, min_b, a.ctypes.data, cap, C.byref(la),
                              b.ctypes.data, cap, C.byref(lb)))
        return a[: la.value].copy(), b[: lb.value].copy()

    # ---- hot path
    def bptt(self, params, act, inputs, targets, weights, h0, loss_scale=1.0,
             clip=3.4028234663852886e38, compute_grads=True, threads=1):
        """bptt_run softmax mode.  Returns dict(loss, positions, h_final,
        g_in_words, g_in_rows (slot order), g_in_dense, g_rec, g_out)."""
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        T, B = inputs.shape
        hf = np.empty((B, H), np.float32)
        nrows = C.c_int64(0)
        gw = np.zeros(T * B, np.uint32)
        gd = np.zeros((T * B, H), np.float32)
        grec = np.zeros((H, H), np.float32)
        gout = np.zeros((V, H), np.float32)
        loss, pos = C.c_double(), C.c_uint64()
        self._check(self._bptt(V, H, act, w_in, w_rec, w_out, T, B,
                               np.ascontiguousarray(inputs, np.uint32),
                               np.ascontiguousarray(targets, np.uint32),
                               np.ascontiguousarray(weights, np.uint8),
                               np.ascontiguousarray(h0, np.float32), loss_scale, clip,
                               int(compute_grads), threads, hf.ctypes.data,
                               C.addressof(nrows), gw.ctypes.data, gd.ctypes.data,
                               grec.ctypes.data, gout.ctypes.data, C.byref(loss),
                               C.byref(pos)))
        r = dict(loss=loss.value, positions=pos.value, h_final=hf)
        if compute_grads:
            n = nrows.value
            dense = np.zeros((V, H), np.float32)
            for s in range(n):
                dense[gw[s]] += gd[s]
            r.update(g_in_words=gw[:n].copy(), g_in_rows=gd[:n].copy(),
                     g_in_dense=dense, g_rec=grec, g_out=gout)
        return r

    def _nce_result(self, V, H, T, B, K1, compute_grads, hf, loss, pos, nin, giw, gid,
                    grec, nout, gow, god):
        r = dict(loss=loss.value, positions=pos.value, h_final=hf)
        if compute_grads:
            n, m = nin.value, nout.value
            din = np.zeros((V, H), np.float32)
            for s_ in range(n):
                din[giw[s_]] += gid[s_]
            dout = np.zeros((V, H), np.float32)
            for s_ in range(m):
                dout[gow[s_]] += god[s_]
            r.update(g_in_words=giw[:n].copy(), g_in_rows=gid[:n].copy(), g_in_dense=din,
                     g_rec=grec, g_out_words=gow[:m].copy(), g_out_rows=god[:m].copy(),
                     g_out=dout)
        return r

    def mt_state(self, seed):
        """std::mt19937_64(seed) state: 312 words + position (uint64[313])."""
        st = np.zeros(313, np.uint64)
        getattr(self.lib, self.prefix + "mt_state")(C.c_uint64(seed), st.ctypes.data_as(_vp))
        return st

    def rmsprop(self, params, state, grads, rho, eps, eta, out_dense=True):
        """rmsprop_update in place on copies; returns (params, state, applied)."""
        w_in, w_rec, w_out = [np.array(x, np.float32, copy=True) for x in params]
        m_rec, m_in, m_out = [np.array(x, np.float32, copy=True) for x in state]
        V, H = w_in.shape
        words = np.ascontiguousarray(grads["g_in_words"], np.uint32)
        rows = np.ascontiguousarray(grads["g_in_rows"], np.float32)
        applied = C.c_int()
        if out_dense:
            gout = np.ascontiguousarray(grads["g_out"], np.float32)
            ow, on = None, 0
        else:
            ow = np.ascontiguousarray(grads["g_out_words"], np.uint32)
            gout = np.ascontiguousarray(grads["g_out_rows"], np.float32)
            on = len(ow)
        self._check(self._rms(V, H, w_in, w_rec, w_out, m_rec, m_in, m_out, rho, eps,
                              eta, len(words), words.ctypes.data, rows.ctypes.data,
                              np.ascontiguousarray(grads["g_rec"], np.float32),
                              int(out_dense), on,
                              None if ow is None else ow.ctypes.data,
                              gout.ctypes.data, C.byref(applied)))
        return (w_in, w_rec, w_out), (m_rec, m_in, m_out), bool(applied.value)

    def sharded_ppl(self, params, act, ids, shards, bos=1):
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        tl, pr, ppl = C.c_double(), C.c_uint64(), C.c_double()
        ids = np.ascontiguousarray(ids, np.uint32)
        self._check(self._sppl(V, H, act, w_in, w_rec, w_out, ids, len(ids), shards,
                               bos, 1, C.byref(tl), C.byref(pr), C.byref(ppl)))
        return dict(total_logprob=tl.value, predicted=pr.value, perplexity=ppl.value)

    def rnn_ppl(self, params, act, ids, bos=1):
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        tl, pr, ppl = C.c_double(), C.c_uint64(), C.c_double()
        ids = np.ascontiguousarray(ids, np.uint32)
        self._check(self._rppl(V, H, act, w_in, w_rec, w_out, ids, len(ids), bos, 1,
                               C.byref(tl), C.byref(pr), C.byref(ppl)))
        return dict(total_logprob=tl.value, predicted=pr.value, perplexity=ppl.value)


    # ---- bottleneck model (compress.hpp:38-415)
    def _bn_fn(self, name, argtypes):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = argtypes
        return f

    def bn_init_uniform(self, V, H, P, seed, rng=0.1):
        e = np.empty((V, P), np.float32)
        u = np.empty((P, H), np.float32)
        w_rec = np.empty((H, H), np.float32)
        d = np.empty((H, P), np.float32)
        f = self._bn_fn("bn_init_uniform", [_i64, _i64, _i64, _u64, C.c_double, _f32p, _f32p,
                                             _f32p, _f32p])
        self._check(f(V, H, P, seed, rng, e, u, w_rec, d))
        return e, u, w_rec, d

    def bn_bptt(self, params, act, inputs, targets, weights, h0, loss_scale=1.0,
                clip=3.4028234663852886e38, compute_grads=True):
        """bptt_run over BottleneckAdapter, softmax mode.  Returns dict(loss,
        positions, h_final, g_e (dense V x P), g_u, g_rec, g_d)."""
        e, u, w_rec, d = params
        V, P = e.shape
        H = w_rec.shape[0]
        T, B = inputs.shape
        hf = np.empty((B, H), np.float32)
        g = [np.zeros(s, np.float32) for s in ((V, P), (P, H), (H, H), (H, P))]
        loss, pos = C.c_double(), C.c_uint64()
        f = self._bn_fn("bn_bptt", [_i64, _i64, _i64, C.c_int, _f32p, _f32p, _f32p, _f32p,
                                    _i64, _i64, _u32p, _u32p, _u8p, _f32p, C.c_double,
                                    C.c_float, C.c_int, _vp, _vp, _vp, _vp, _vp,
                                    C.POINTER(C.c_double), C.POINTER(C.c_uint64)])
        self._check(f(V, H, P, act, e, u, w_rec, d, T, B,
                      np.ascontiguousarray(inputs, np.uint32),
                      np.ascontiguousarray(targets, np.uint32),
                      np.ascontiguousarray(weights, np.uint8),
                      np.ascontiguousarray(h0, np.float32), loss_scale, clip,
                      int(compute_grads), hf.ctypes.data, *(x.ctypes.data for x in g),
                      C.byref(loss), C.byref(pos)))
        r = dict(loss=loss.value, positions=pos.value, h_final=hf)
        if compute_grads:
            r.update(g_e=g[0], g_u=g[1], g_rec=g[2], g_d=g[3])
        return r

    def bn_update(self, params, state, grads, rho, eps, eta):
        """bottleneck_update on copies; state = (m_e, m_u, m_rec, m_d)."""
        p = [np.array(x, np.float32, copy=True) for x in params]
        m = [np.array(x, np.float32, copy=True) for x in state]
        V, P = p[0].shape
        H = p[2].shape[0]
        applied = C.c_int()
        f = self._bn_fn("bn_update", [_i64, _i64, _i64] + [_f32p] * 8 +
                        [C.c_double] * 3 + [_f32p] * 4 + [C.POINTER(C.c_int)])
        gs = [np.ascontiguousarray(grads[k], np.float32) for k in ("g_e", "g_u", "g_rec", "g_d")]
        self._check(f(V, H, P, *p, *m, rho, eps, eta, *gs, C.byref(applied)))
        return tuple(p), tuple(m), bool(applied.value)

    def _bn_nce_result(self, V, H, P, compute_grads, hf, loss, pos, ne, gew, ged, g):
        r = dict(loss=loss.value, positions=pos.value, h_final=hf)
        if compute_grads:
            n = ne.value
            dense = np.zeros((V, P), np.float32)
            for s_ in range(n):
                dense[gew[s_]] += ged[s_]
            r.update(g_e_words=gew[:n].copy(), g_e_rows=ged[:n].copy(), g_e=dense, g_u=g[0],
                     g_rec=g[1], g_d=g[2])
        return r

    def bn_update_sparse(self, params, state, grads, rho, eps, eta):
        """bottleneck_update with the sparse embedding gradient (NCE mode)."""
        p = [np.array(x, np.float32, copy=True) for x in params]
        m = [np.array(x, np.float32, copy=True) for x in state]
        V, P = p[0].shape
        H = p[2].shape[0]
        applied = C.c_int()
        f = self._bn_fn("bn_update_sparse", [_i64, _i64, _i64] + [_f32p] * 8 +
                        [C.c_double] * 3 + [_i64, _vp, _vp] + [_f32p] * 3 +
                        [C.POINTER(C.c_int)])
        words = np.ascontiguousarray(grads["g_e_words"], np.uint32)
        rows = np.ascontiguousarray(grads["g_e_rows"], np.float32)
        gs = [np.ascontiguousarray(grads[k], np.float32) for k in ("g_u", "g_rec", "g_d")]
        self._check(f(V, H, P, *p, *m, rho, eps, eta, len(words), words.ctypes.data,
                      rows.ctypes.data, *gs, C.byref(applied)))
        return tuple(p), tuple(m), bool(applied.value)

    def ln_z_samples(self, params, act, ids, count):
        """ln_z_samples (eval.hpp:805-857) -> float64 array."""
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        ids = np.ascontiguousarray(ids, np.uint32)
        out = np.empty(count, np.float64)
        ns = C.c_int64()
        if self.prefix == "ref_":
            stats = np.zeros(6, np.float64)
            f = self.lib.ref_ln_z_samples
            f.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _u32p, _i64, _i64, _vp,
                          C.POINTER(C.c_int64), _vp]
            self._check(f(V, H, act, w_in, w_rec, w_out, ids, len(ids), count, out.ctypes.data,
                          C.byref(ns), stats.ctypes.data))
            self.last_drift_stats = stats
        else:
            f = self.lib.orc_ln_z_samples
            f.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _u32p, _i64, _i64, _vp,
                          C.POINTER(C.c_int64)]
            self._check(f(V, H, act, w_in, w_rec, w_out, ids, len(ids), count, out.ctypes.data,
                          C.byref(ns)))
        return out[: ns.value].copy()

    def bn_sharded_ppl(self, params, act, ids, shards, bos=1):
        e, u, w_rec, d = params
        V, P = e.shape
        H = w_rec.shape[0]
        tl, pr, ppl = C.c_double(), C.c_uint64(), C.c_double()
        ids = np.ascontiguousarray(ids, np.uint32)
        f = self._bn_fn("bn_sharded_ppl", [_i64, _i64, _i64, C.c_int, _f32p, _f32p, _f32p,
                                           _f32p, _u32p, _i64, C.c_int, C.c_uint32,
                                           C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_double)])
        self._check(f(V, H, P, act, e, u, w_rec, d, ids, len(ids), shards, bos,
                      C.byref(tl), C.byref(pr), C.byref(ppl)))
        return dict(total_logprob=tl.value, predicted=pr.value, perplexity=ppl.value)


    def bn_train(self, cfg, params, train_ids, valid_ids):
        """Trainer<BottleneckTraits>::train (trainer.hpp:178-270, 350-410;
        compress.hpp:389-415), softmax mode, restated over this backend's
        bn_bptt / bn_update / bn_sharded_ppl (a Python loop: small cases).
        Returns dict(logs [n x 7] (seconds / tokens_per_sec zero),
        initial_ppl, params, opt, cursors, hidden)."""
        e, u, w_rec, d = [np.array(x, np.float32, copy=True) for x in params]
        V, P = e.shape
        H = cfg.nstate
        tr = np.ascontiguousarray(train_ids, np.uint32)
        va = np.ascontiguousarray(valid_ids, np.uint32)
        if cfg.valid_limit > 0 and len(va) > cfg.valid_limit:
            va = va[: cfg.valid_limit]
        L, B, T = len(tr), cfg.minibatch, cfg.unroll
        N = cfg.noffset * B
        cur = np.array([i * L // N for i in range(N)], np.int64)
        a0 = np.float32(0.5) if cfg.act == 0 else np.float32(0.0)
        hidden = np.full((N, H), a0, np.float32)
        state = (np.zeros(V, np.float32), np.zeros((P, H), np.float32),
                 np.zeros((H, H), np.float32), np.zeros((H, P), np.float32))
        prm = (e, u, w_rec, d)
        nce = cfg.mode == 0
        if nce:
            # NoiseModel::from_stream over the non-bos training tokens; the
            # trainer's rng seeded with cfg.seed (trainer.hpp:184, 207-209)
            counts = np.bincount(tr[tr != 1], minlength=V).astype(np.float64)
            noise = self.noise_build(counts, cfg.nce_k, cfg.noise_floor) \
                if hasattr(self, "noise_build") else None
            st_rng = self.mt_state(cfg.seed)

        def validate():
            return self.bn_sharded_ppl(prm, cfg.act, va, cfg.valid_shards)["perplexity"]

        initial = validate()
        best, bad, eta, epoch, logs = initial, 0, cfg.eta, 0, []
        rounds = (L + N * T - 1) // (N * T)
        tt = np.arange(T)[:, None]
        while epoch < cfg.max_epochs and bad < 2:
            loss_sum, windows, skipped = 0.0, 0, 0
            for _ in range(rounds):
                for g in range(cfg.noffset):
                    s0 = g * B
                    pos = cur[None, s0:s0 + B] + tt
                    x = tr[pos % L]
                    y = tr[(pos + 1) % L]
                    w = (y != 1).astype(np.uint8)
                    if nce:
                        r = self.bn_bptt_nce(prm, cfg.act, x, y, w, hidden[s0:s0 + B],
                                             1.0 / (B * T), cfg.clip, noise, st_rng)
                    else:
                        r = self.bn_bptt(prm, cfg.act, x, y, w, hidden[s0:s0 + B],
                                         1.0 / (B * T), cfg.clip)
                    loss_sum += r["loss"]
                    windows += 1
                    upd = self.bn_update_sparse if nce else self.bn_update
                    prm, state, ok = upd(prm, state, r, cfg.rho, cfg.eps, eta)
                    skipped += 0 if ok else 1
                    hidden[s0:s0 + B] = r["h_final"]
                    cur[s0:s0 + B] += T
                    wrap = cur[s0:s0 + B] >= L
                    cur[s0:s0 + B][wrap] -= L
                    hidden[s0:s0 + B][wrap] = a0
            ppl = validate()
            epoch += 1
            logs.append([epoch, loss_sum / windows if windows else 0.0, ppl, eta, 0.0, 0.0,
                         skipped])
            if ppl > cfg.divergence_factor * initial:
                raise OracleError(2, "trainer: diverged")
            if ppl < best:
                best, bad = ppl, 0
            else:
                bad += 1
                eta *= 0.5
        return dict(logs=np.array(logs, np.float64), initial_ppl=initial, params=prm, opt=state,
                    cursors=cur, hidden=hidden, rng=st_rng if nce else self.mt_state(cfg.seed))


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


class Orc(_Backend):
    """The C restatement (oracle/desklm_oracle.c)."""

    prefix = "orc_"
    so_path = ORC_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        self._slp = L.orc_sharded_logprobs
        self._slp.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _u32p, _i64,
                              C.c_int, C.c_uint32, _vp, _i64, C.POINTER(C.c_int64),
                              C.POINTER(C.c_int64), C.POINTER(C.c_double),
                              C.POINTER(C.c_uint64)]
        self._wb = L.orc_window_build
        self._wb.argtypes = [_u32p, _i64, _i64p, _i64, _i64, _i64, C.c_uint32,
                             _u32p, _u32p, _u8p]
        self._train = L.orc_train
        self._train.argtypes = [C.POINTER(TrainConfig), _i64, _f32p, _f32p, _f32p,
                                _u32p, _i64, _u32p, _i64, C.c_int, _f32p, _f32p,
                                _f32p, _i64p, _f32p, _f64p, C.POINTER(C.c_int),
                                C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_double), C.POINTER(C.c_int),
                                C.POINTER(C.c_int)]

    def sharded_logprobs(self, params, act, ids, shards, bos=1):
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        ids = np.ascontiguousarray(ids, np.uint32)
        S, steps = C.c_int64(), C.c_int64()
        tl, pr = C.c_double(), C.c_uint64()
        n = len(ids)
        Smax = min(shards, n // 2)
        cap = (n // max(Smax, 1) + 2) * max(Smax, 1)
        out = np.empty(cap, np.float64)
        self._check(self._slp(V, H, act, w_in, w_rec, w_out, ids, n, shards, bos,
                              out.ctypes.data, cap, C.byref(S), C.byref(steps),
                              C.byref(tl), C.byref(pr)))
        return out[: S.value * steps.value].reshape(steps.value, S.value).copy()

    def window_build(self, ids, cursors, s0, B, T, bos=1):
        ids = np.ascontiguousarray(ids, np.uint32)
        cur = np.ascontiguousarray(cursors, np.int64)
        x = np.empty((T, B), np.uint32)
        y = np.empty((T, B), np.uint32)
        w = np.empty((T, B), np.uint8)
        self._wb(ids, len(ids), cur, s0, B, T, bos, x, y, w)
        return x, y, w

    def train(self, cfg: TrainConfig, params, train_ids, valid_ids, run=True):
        w_in, w_rec, w_out = [np.array(x, np.float32, copy=True) for x in params]
        V, H = w_in.shape
        N = cfg.noffset * cfg.minibatch
        m_rec = np.zeros((H, H), np.float32)
        m_in = np.zeros(V, np.float32)
        m_out = np.zeros(V, np.float32)
        cur = np.zeros(N, np.int64)
        hid = np.zeros((N, H), np.float32)
        logs = np.zeros((max(cfg.max_epochs, 1), 7), np.float64)
        nl, bad, ep = C.c_int(), C.c_int(), C.c_int()
        ini, eta, best = C.c_double(), C.c_double(), C.c_double()
        tr = np.ascontiguousarray(train_ids, np.uint32)
        va = np.ascontiguousarray(valid_ids, np.uint32)
        rc = self._train(C.byref(cfg), V, w_in, w_rec, w_out, tr, len(tr), va, len(va),
                         int(run), m_rec, m_in, m_out, cur, hid, logs, C.byref(nl),
                         C.byref(ini), C.byref(eta), C.byref(best), C.byref(bad),
                         C.byref(ep))
        if rc not in (0,):
            raise OracleError(rc, "orc_train")
        rng = np.zeros(313, np.uint64)
        self.lib.orc_last_train_rng(rng.ctypes.data_as(C.c_void_p))
        return dict(params=(w_in, w_rec, w_out), opt=(m_rec, m_in, m_out),
                    cursors=cur, hidden=hid, logs=logs[: nl.value].copy(),
                    initial_ppl=ini.value, eta=eta.value, best_ppl=best.value,
                    bad_epochs=bad.value, epoch=ep.value, rng_state=rng)


    def noise_build(self, counts, k, floor=1e-8):
        """NoiseModel + AliasSampler tables (nce.hpp:41-66, rng.hpp:54-89)."""
        counts = np.ascontiguousarray(counts, np.float64)
        V = len(counts)
        q, lnkq, prob = (np.empty(V, np.float64) for _ in range(3))
        alias = np.empty(V, np.uint32)
        f = self.lib.orc_noise_build
        f.argtypes = [_i64, _vp, C.c_int, C.c_double, _vp, _vp, _vp, _vp]
        self._check(f(V, counts.ctypes.data, int(k), float(floor), q.ctypes.data,
                      lnkq.ctypes.data, prob.ctypes.data, alias.ctypes.data))
        return dict(k=int(k), q=q, ln_kq=lnkq, prob=prob, alias=alias)

    def noise_sample(self, noise, rng, n):
        out = np.empty(n, np.uint32)
        f = self.lib.orc_noise_sample
        f.argtypes = [_i64, _vp, _vp, _vp, _i64, _vp]
        self._check(f(len(noise["prob"]), noise["prob"].ctypes.data, noise["alias"].ctypes.data,
                      rng.ctypes.data, n, out.ctypes.data))
        return out

    def bn_bptt_nce(self, params, act, inputs, targets, weights, h0, loss_scale, clip, noise,
                    rng, compute_grads=True):
        """bptt_run over the bottleneck adapter in NCE mode; rng advanced in place."""
        e, u, w_rec, d = params
        V, P = e.shape
        H = w_rec.shape[0]
        T, B = inputs.shape
        k = noise["k"]
        hf = np.empty((B, H), np.float32)
        ne = C.c_int64(0)
        gew = np.zeros(T * B * (k + 2), np.uint32)
        ged = np.zeros((T * B * (k + 2), P), np.float32)
        g = [np.zeros(sh, np.float32) for sh in ((P, H), (H, H), (H, P))]
        loss, pos = C.c_double(), C.c_uint64()
        f = self.lib.orc_bn_bptt_nce
        f.argtypes = [_i64, _i64, _i64, C.c_int] + [_f32p] * 4 + [_i64, _i64, _u32p, _u32p,
                                                                   _u8p, _f32p, C.c_double,
                                                                   C.c_float, C.c_int, C.c_int] + \
            [_vp] * 11 + [C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        self._check(f(V, H, P, act, e, u, w_rec, d, T, B,
                      np.ascontiguousarray(inputs, np.uint32),
                      np.ascontiguousarray(targets, np.uint32),
                      np.ascontiguousarray(weights, np.uint8),
                      np.ascontiguousarray(h0, np.float32), loss_scale, clip,
                      int(compute_grads), k, noise["ln_kq"].ctypes.data,
                      noise["prob"].ctypes.data, noise["alias"].ctypes.data, rng.ctypes.data,
                      hf.ctypes.data, C.addressof(ne), gew.ctypes.data, ged.ctypes.data,
                      *(x.ctypes.data for x in g), C.byref(loss), C.byref(pos)))
        return self._bn_nce_result(V, H, P, compute_grads, hf, loss, pos, ne, gew, ged, g)

    def bptt_nce(self, params, act, inputs, targets, weights, h0, loss_scale, clip, noise, rng,
                 compute_grads=True):
        """bptt_run NCE mode (backprop.hpp:126-156); rng (uint64[313]) is
        advanced in place.  Returns the bptt dict plus g_out_words /
        g_out_rows (sparse, slot order) and the draws."""
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        T, B = inputs.shape
        k = noise["k"]
        K1 = k + 1
        hf = np.empty((B, H), np.float32)
        nin, nout = C.c_int64(0), C.c_int64(0)
        giw = np.zeros(T * B, np.uint32)
        gid = np.zeros((T * B, H), np.float32)
        grec = np.zeros((H, H), np.float32)
        gow = np.zeros(T * B * K1, np.uint32)
        god = np.zeros((T * B * K1, H), np.float32)
        draws = np.zeros(T * B * k, np.uint32)
        loss, pos = C.c_double(), C.c_uint64()
        f = self.lib.orc_bptt_nce
        f.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _i64, _i64, _u32p, _u32p,
                      _u8p, _f32p, C.c_double, C.c_float, C.c_int, C.c_int, _vp, _vp, _vp,
                      _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                      C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        self._check(f(V, H, act, w_in, w_rec, w_out, T, B,
                      np.ascontiguousarray(inputs, np.uint32),
                      np.ascontiguousarray(targets, np.uint32),
                      np.ascontiguousarray(weights, np.uint8),
                      np.ascontiguousarray(h0, np.float32), loss_scale, clip,
                      int(compute_grads), k, noise["ln_kq"].ctypes.data,
                      noise["prob"].ctypes.data, noise["alias"].ctypes.data, rng.ctypes.data,
                      hf.ctypes.data, C.addressof(nin), giw.ctypes.data, gid.ctypes.data,
                      grec.ctypes.data, C.addressof(nout), gow.ctypes.data, god.ctypes.data,
                      draws.ctypes.data, C.byref(loss), C.byref(pos)))
        r = self._nce_result(V, H, T, B, K1, compute_grads, hf, loss, pos, nin, giw, gid, grec,
                             nout, gow, god)
        r["noise"] = draws[:r["positions"] * k].copy()
        return r


class Ref(_Backend):
    """The reference itself (oracle/_ref/libdesklm_ref.so)."""

    prefix = "ref_"
    so_path = REF_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        self._slp = L.ref_sharded_logprobs
        self._slp.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _u32p, _i64,
                              C.c_int, C.c_uint32, _vp, _i64, C.POINTER(C.c_int64),
                              C.POINTER(C.c_int64)]
        self._train = L.ref_train
        self._train.argtypes = [C.POINTER(TrainConfig), _i64, _f32p, _f32p, _f32p,
                                _u32p, _i64, _u32p, _i64, C.c_int, _vp, _u64,
                                C.POINTER(C.c_uint64), _f64p, C.POINTER(C.c_int),
                                C.POINTER(C.c_double)]
        self._wp = L.ref_write_params
        self._wp.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _vp, _u64,
                             C.POINTER(C.c_uint64)]
        self._wr = L.ref_write_rmsprop
        self._wr.argtypes = [_i64, _i64, C.c_double, C.c_double, _f32p, _f32p, _f32p,
                             _vp, _u64, C.POINTER(C.c_uint64)]
        self._rescore = L.ref_rescore
        self._rescore.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p,
                                  C.c_char_p, C.c_double, C.c_double, C.c_int, _vp,
                                  _u64, C.POINTER(C.c_uint64)]

    def bn_train_native(self, cfg, params, train_ids, valid_ids, run=True):
        """The reference's own Trainer<BottleneckTraits>: (rtrn_bytes, logs, initial)."""
        e, u, w_rec, d = params
        V, P = e.shape
        H = cfg.nstate
        tr = np.ascontiguousarray(train_ids, np.uint32)
        va = np.ascontiguousarray(valid_ids, np.uint32)
        N = cfg.noffset * cfg.minibatch
        cap = 16384 + 8 * N + 4 * N * H + 8 * (V * P + 2 * P * H + H * H + 2 * H * P) + \
            64 * V + 8 * V
        buf = np.zeros(cap, np.uint8)
        ln = C.c_uint64()
        logs = np.zeros((max(cfg.max_epochs, 1), 7), np.float64)
        nl = C.c_int()
        ini = C.c_double()
        f = self.lib.ref_bn_train
        f.argtypes = [C.POINTER(TrainConfig), _i64, _i64, _f32p, _f32p, _f32p, _f32p, _u32p,
                      _i64, _u32p, _i64, C.c_int, _vp, _u64, C.POINTER(C.c_uint64), _f64p,
                      C.POINTER(C.c_int), C.POINTER(C.c_double)]
        self._check(f(C.byref(cfg), V, P, e, u, w_rec, d, tr, len(tr), va, len(va), int(run),
                      buf.ctypes.data, cap, C.byref(ln), logs, C.byref(nl), C.byref(ini)))
        return bytes(buf[: ln.value]), logs[: nl.value].copy(), ini.value

    def ngram_query(self, train, V, order, contexts, words, k, eval_ids):
        """count_ngrams + estimate_kn, then logprob / shortlist per query and
        ngram_perplexity_full of eval_ids."""
        ctx_len = max(1, max((len(c) for c in contexts), default=1))
        nq = len(words)
        ctx = np.full((nq, ctx_len), -1, np.int64)
        for i, c in enumerate(contexts):
            if len(c):
                ctx[i, ctx_len - len(c):] = c
        words = np.ascontiguousarray(words, np.uint32)
        logp = np.empty(nq, np.float64)
        sl = np.empty((nq, k), np.uint32)
        ppl = np.empty(3, np.float64)
        tr = np.ascontiguousarray(train, np.uint32)
        ev = np.ascontiguousarray(eval_ids, np.uint32)
        f = self.lib.ref_ngram_query
        f.argtypes = [_u32p, _i64, _i64, C.c_int, _i64, C.c_int, _vp, _u32p, _vp, C.c_int, _vp,
                      _u32p, _i64, _vp]
        self._check(f(tr, len(tr), V, order, nq, ctx_len, ctx.ctypes.data, words,
                      logp.ctypes.data, k, sl.ctypes.data, ev, len(ev), ppl.ctypes.data))
        return logp, [list(r[r != 0xffffffff]) for r in sl], ppl

    def interp_terms(self, params, act, Vf, train, order, eval_ids):
        """interpolation_terms + tune_lambda (RNN vocabulary make_vocab(Vr),
        n-gram vocabulary make_vocab(Vf))."""
        w_in, w_rec, w_out = params
        Vr, H = w_in.shape
        tr = np.ascontiguousarray(train, np.uint32)
        ev = np.ascontiguousarray(eval_ids, np.uint32)
        a = np.empty(len(ev), np.float64)
        b = np.empty(len(ev), np.float64)
        nt = C.c_int64()
        lp = np.empty(2, np.float64)
        f = self.lib.ref_interp_terms
        f.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _i64, _u32p, _i64, C.c_int,
                      _u32p, _i64, _vp, _vp, C.POINTER(C.c_int64), _vp]
        self._check(f(Vr, H, act, w_in, w_rec, w_out, Vf, tr, len(tr), order, ev, len(ev),
                      a.ctypes.data, b.ctypes.data, C.byref(nt), lp.ctypes.data))
        n = nt.value
        return a[:n].copy(), b[:n].copy(), float(lp[0]), float(lp[1])

    def hit_rate(self, params, act, train, order, eval_ids, shortlist_k, top_k, kind):
        """hit_rate with RnnHitScorer (kind 0) or NgramHitScorer (kind 1)."""
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        tr = np.ascontiguousarray(train, np.uint32)
        ev = np.ascontiguousarray(eval_ids, np.uint32)
        pos, hits = C.c_uint64(), C.c_uint64()
        f = self.lib.ref_hit_rate
        f.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _u32p, _i64, C.c_int, _u32p,
                      _i64, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64),
                      C.POINTER(C.c_uint64)]
        self._check(f(V, H, act, w_in, w_rec, w_out, tr, len(tr), order, ev, len(ev),
                      shortlist_k, top_k, kind, C.byref(pos), C.byref(hits)))
        return pos.value, hits.value

    def gen_corpus(self, gen_seed, train_tokens, train_seed, valid_tokens, valid_seed, V):
        """TextGenerator(GenConfig{}, gen_seed) -> normalize -> build_vocab
        -> encode: (train ids, valid ids)."""
        ct, cv = int(train_tokens * 1.5) + 1000, int(valid_tokens * 1.5) + 1000
        a = np.empty(ct, np.uint32)
        b = np.empty(cv, np.uint32)
        na, nb = C.c_int64(), C.c_int64()
        f = self.lib.ref_gen_corpus
        f.argtypes = [_u64, _i64, _u64, _i64, _u64, _i64, _vp, _i64, C.POINTER(C.c_int64), _vp,
                      _i64, C.POINTER(C.c_int64)]
        self._check(f(gen_seed, train_tokens, train_seed, valid_tokens, valid_seed, V,
                      a.ctypes.data, ct, C.byref(na), b.ctypes.data, cv, C.byref(nb)))
        return a[: min(na.value, ct)].copy(), b[: min(nb.value, cv)].copy()

    def bn_quantize(self, params, bits, act=0):
        """quantize_model + write_quantized (RNQZ bytes) and the dequantized
        parameters of read_quantized + dequantize_model."""
        e, u, w_rec, d = params
        V, P = e.shape
        H = w_rec.shape[0]
        f = self.lib.ref_bn_quantize
        f.argtypes = [_i64, _i64, _i64, C.c_int] + [_f32p] * 4 + [C.c_int, _vp, _u64,
                                                                  C.POINTER(C.c_uint64)] + \
            [_f32p] * 4
        cap = (V * P + 2 * P * H + H * H) * 2 + 64 * V + 4096
        buf = np.zeros(cap, np.uint8)
        ln = C.c_uint64()
        out = [np.empty(s_, np.float32) for s_ in ((V, P), (P, H), (H, H), (H, P))]
        self._check(f(V, H, P, act, e, u, w_rec, d, int(bits), buf.ctypes.data, cap,
                      C.byref(ln), *out))
        return bytes(buf[: ln.value]), tuple(out)

    def bn_write(self, params, state, rho, eps, act=0):
        """write_bottleneck (RNBL, vocabulary make_vocab(V)) and
        write_bottleneck_opt (RBOP) bytes."""
        e, u, w_rec, d = params
        V, P = e.shape
        H = w_rec.shape[0]
        f = self.lib.ref_bn_write
        f.argtypes = [_i64, _i64, _i64, C.c_int] + [_f32p] * 4 + [C.c_double] * 2 + \
            [_f32p] * 4 + [_vp, _u64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        cap = 4 * (2 * V * P + 2 * P * H + 2 * H * H + 2 * H * P + V) + 32 * V + 4096
        buf = np.zeros(cap, np.uint8)
        lp, ln = C.c_uint64(), C.c_uint64()
        m = [np.ascontiguousarray(x, np.float32) for x in state]
        self._check(f(V, H, P, act, e, u, w_rec, d, rho, eps, *m, buf.ctypes.data, cap,
                      C.byref(lp), C.byref(ln)))
        b = bytes(buf[: ln.value])
        return b[: lp.value], b[lp.value:]

    def sharded_logprobs(self, params, act, ids, shards, bos=1):
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        ids = np.ascontiguousarray(ids, np.uint32)
        n = len(ids)
        Smax = min(shards, n // 2)
        cap = (n // max(Smax, 1) + 2) * max(Smax, 1)
        out = np.empty(cap, np.float64)
        S, steps = C.c_int64(), C.c_int64()
        self._check(self._slp(V, H, act, w_in, w_rec, w_out, ids, n, shards, bos,
                              out.ctypes.data, cap, C.byref(S), C.byref(steps)))
        return out[: S.value * steps.value].reshape(steps.value, S.value).copy()

    def train(self, cfg: TrainConfig, params, train_ids, valid_ids, run=True):
        """Returns (rtrn_bytes, logs[n,7], initial_ppl)."""
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        tr = np.ascontiguousarray(train_ids, np.uint32)
        va = np.ascontiguousarray(valid_ids, np.uint32)
        N = cfg.noffset * cfg.minibatch
        cap = 16384 + 8 * N + 4 * N * H + 8 * (2 * V * H + H * H) + 64 * V + 8 * V
        buf = np.zeros(cap, np.uint8)
        ln = C.c_uint64()
        logs = np.zeros((max(cfg.max_epochs, 1), 7), np.float64)
        nl = C.c_int()
        ini = C.c_double()
        self._check(self._train(C.byref(cfg), V, w_in, w_rec, w_out, tr, len(tr), va,
                                len(va), int(run), buf.ctypes.data, cap, C.byref(ln),
                                logs, C.byref(nl), C.byref(ini)))
        return bytes(buf[: ln.value]), logs[: nl.value].copy(), ini.value

    def write_params(self, params, act=0):
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        ln = C.c_uint64()
        self._wp(V, H, act, w_in, w_rec, w_out, None, 0, C.byref(ln))
        buf = np.zeros(ln.value, np.uint8)
        self._check(self._wp(V, H, act, w_in, w_rec, w_out, buf.ctypes.data, ln.value,
                             C.byref(ln)))
        return bytes(buf)

    def write_rmsprop(self, V, H, rho, eps, state):
        m_rec, m_in, m_out = [np.ascontiguousarray(x, np.float32) for x in state]
        ln = C.c_uint64()
        self._wr(V, H, rho, eps, m_rec, m_in, m_out, None, 0, C.byref(ln))
        buf = np.zeros(ln.value, np.uint8)
        self._check(self._wr(V, H, rho, eps, m_rec, m_in, m_out, buf.ctypes.data,
                             ln.value, C.byref(ln)))
        return bytes(buf)

    def rescore(self, params, act, nbest_text, lm_scale=1.0, wip=0.0, fast=False):
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        cap = 4 * len(nbest_text) + 1 << 16
        buf = C.create_string_buffer(cap)
        ln = C.c_uint64()
        self._check(self._rescore(V, H, act, w_in, w_rec, w_out, nbest_text.encode(),
                                  lm_scale, wip, int(fast), C.addressof(buf), cap,
                                  C.byref(ln)))
        return buf.value.decode()


    def noise_sample(self, counts, k, floor, rng, n):
        """n draws of NoiseModel(counts, k, floor).sample (rng advanced in
        place) and its ln(k q) table."""
        counts = np.ascontiguousarray(counts, np.float64)
        V = len(counts)
        out = np.empty(n, np.uint32)
        lnkq = np.empty(V, np.float64)
        f = self.lib.ref_noise_sample
        f.argtypes = [_i64, _vp, C.c_int, C.c_double, _vp, _i64, _vp, _vp]
        self._check(f(V, counts.ctypes.data, int(k), float(floor), rng.ctypes.data, n,
                      out.ctypes.data, lnkq.ctypes.data))
        return out, lnkq

    def bn_bptt_nce(self, params, act, inputs, targets, weights, h0, loss_scale, clip, counts,
                    k, floor, rng, compute_grads=True):
        e, u, w_rec, d = params
        V, P = e.shape
        H = w_rec.shape[0]
        T, B = inputs.shape
        counts = np.ascontiguousarray(counts, np.float64)
        hf = np.empty((B, H), np.float32)
        ne = C.c_int64(0)
        gew = np.zeros(T * B * (k + 2), np.uint32)
        ged = np.zeros((T * B * (k + 2), P), np.float32)
        g = [np.zeros(sh, np.float32) for sh in ((P, H), (H, H), (H, P))]
        loss, pos = C.c_double(), C.c_uint64()
        f = self.lib.ref_bn_bptt_nce
        f.argtypes = [_i64, _i64, _i64, C.c_int] + [_f32p] * 4 + [_i64, _i64, _u32p, _u32p,
                                                                   _u8p, _f32p, C.c_double,
                                                                   C.c_float, C.c_int, _vp,
                                                                   C.c_int, C.c_double] + \
            [_vp] * 8 + [C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        self._check(f(V, H, P, act, e, u, w_rec, d, T, B,
                      np.ascontiguousarray(inputs, np.uint32),
                      np.ascontiguousarray(targets, np.uint32),
                      np.ascontiguousarray(weights, np.uint8),
                      np.ascontiguousarray(h0, np.float32), loss_scale, clip,
                      int(compute_grads), counts.ctypes.data, int(k), float(floor),
                      rng.ctypes.data, hf.ctypes.data, C.addressof(ne), gew.ctypes.data,
                      ged.ctypes.data, *(x.ctypes.data for x in g), C.byref(loss),
                      C.byref(pos)))
        return self._bn_nce_result(V, H, P, compute_grads, hf, loss, pos, ne, gew, ged, g)

    def bptt_nce(self, params, act, inputs, targets, weights, h0, loss_scale, clip, counts, k,
                 floor, rng, compute_grads=True):
        w_in, w_rec, w_out = params
        V, H = w_in.shape
        T, B = inputs.shape
        K1 = k + 1
        counts = np.ascontiguousarray(counts, np.float64)
        hf = np.empty((B, H), np.float32)
        nin, nout = C.c_int64(0), C.c_int64(0)
        giw = np.zeros(T * B, np.uint32)
        gid = np.zeros((T * B, H), np.float32)
        grec = np.zeros((H, H), np.float32)
        gow = np.zeros(T * B * K1, np.uint32)
        god = np.zeros((T * B * K1, H), np.float32)
        loss, pos = C.c_double(), C.c_uint64()
        f = self.lib.ref_bptt_nce
        f.argtypes = [_i64, _i64, C.c_int, _f32p, _f32p, _f32p, _i64, _i64, _u32p, _u32p,
                      _u8p, _f32p, C.c_double, C.c_float, C.c_int, _vp, C.c_int, C.c_double,
                      _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                      C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        self._check(f(V, H, act, w_in, w_rec, w_out, T, B,
                      np.ascontiguousarray(inputs, np.uint32),
                      np.ascontiguousarray(targets, np.uint32),
                      np.ascontiguousarray(weights, np.uint8),
                      np.ascontiguousarray(h0, np.float32), loss_scale, clip,
                      int(compute_grads), counts.ctypes.data, int(k), float(floor),
                      rng.ctypes.data, hf.ctypes.data, C.addressof(nin), giw.ctypes.data,
                      gid.ctypes.data, grec.ctypes.data, C.addressof(nout), gow.ctypes.data,
                      god.ctypes.data, C.byref(loss), C.byref(pos)))
        return self._nce_result(V, H, T, B, K1, compute_grads, hf, loss, pos, nin, giw, gid,
                                grec, nout, gow, god)


def have_ref() -> bool:
    return os.path.exists(REF_SO)
