"""Byte-exact desklm file formats (little-endian), written fresh from the
reference's documented layouts:

* RNLM model     -- rnn.hpp:263-308   (W_out stored H x V, transposed from memory)
* ROPT optimiser -- rmsprop.hpp:137-170 (40-byte header + m_rec, m_in, m_out)
* RTRN trainer   -- trainer.hpp:274-341 + config echo :412-457
* LE primitives  -- util.hpp:84-162
"""
from __future__ import annotations

import io
from dataclasses import dataclass
import struct

import numpy as np

from ._lib import DataError

RNN_FORMAT_VERSION = 1
RMSPROP_FORMAT_VERSION = 1
TRAINER_FORMAT_VERSION = 1
RMSPROP_HEADER_BYTES = 4 + 4 + 8 + 8 + 8 + 8


# ------------------------------------------------------------ primitives
class Reader:
    def __init__(self, data: bytes):
        self.b = memoryview(data)
        self.i = 0

    def take(self, n: int) -> bytes:
        if self.i + n > len(self.b):
            raise DataError("unexpected end of file")
        out = bytes(self.b[self.i:self.i + n])
        self.i += n
        return out

    def u8(self): return self.take(1)[0]
    def u32(self): return struct.unpack("<I", self.take(4))[0]
    def u64(self): return struct.unpack("<Q", self.take(8))[0]
    def f64(self): return struct.unpack("<d", self.take(8))[0]

    def f32s(self, n: int) -> np.ndarray:
        return np.frombuffer(self.take(4 * n), dtype="<f4").astype(np.float32)

    def string(self) -> str:
        n = self.u64()
        return self.take(n).decode("utf-8", errors="surrogateescape")

    def magic(self, m: str, what: str):
        if self.i + 4 > len(self.b) or bytes(self.b[self.i:self.i + 4]) != m.encode():
            raise DataError(f"bad magic, not a {what} file")
        self.i += 4


def _u8(v): return struct.pack("<B", v)
def _u32(v): return struct.pack("<I", v)
def _u64(v): return struct.pack("<Q", v)
def _f64(v): return struct.pack("<d", v)


def _str(s: str) -> bytes:
    b = s.encode("utf-8", errors="surrogateescape")
    return _u64(len(b)) + b


# ------------------------------------------------- vocabulary / id streams
SPECIALS = ("<unk>", "<s>", "</s>")  # ids 0, 1, 2 (corpus.hpp:54-74)


def read_vocab(text: str):
    """Vocabulary::read (corpus.hpp:96-104): one word per line (a trailing
    CR is dropped); must start with <unk>, <s>, </s>."""
    words = text.split("\n")
    if words and words[-1] == "":
        words.pop()
    words = [w[:-1] if w.endswith("\r") else w for w in words]
    if len(words) < 3 or tuple(words[:3]) != SPECIALS:
        raise DataError("vocabulary must start with <unk>, <s>, </s>")
    return words


def write_vocab(words) -> str:
    """Vocabulary::write (corpus.hpp:92-94)."""
    return "".join(w + "\n" for w in words)


def read_id_stream(text: str, vocab_size: int) -> np.ndarray:
    """read_id_stream (corpus.hpp:264-279): whitespace-separated decimal ids,
    each < vocab_size."""
    out = []
    line = 1
    for tok in text.split():
        try:
            v = int(tok)
            if v < 0:
                raise ValueError
        except ValueError:
            raise DataError(f"id stream: not a number: {tok} (line {line})")
        if v >= vocab_size:
            raise DataError(f"id stream: id out of range: {tok}")
        out.append(v)
    return np.array(out, np.uint32)


def write_id_stream(ids, eos_id: int = 2) -> str:
    """write_id_stream (corpus.hpp:256-262): one sentence per line."""
    return "".join(f"{int(i)}{chr(10) if int(i) == eos_id else ' '}" for i in ids)


# ------------------------------------------------------------------ RNLM
def write_params(params, vocab_words, act: int = 0) -> bytes:
    """rnn.hpp:263-285."""
    w_in, w_rec, w_out = params
    V, H = w_in.shape
    out = io.BytesIO()
    out.write(b"RNLM" + _u32(RNN_FORMAT_VERSION) + _u64(V) + _u64(H) + _u8(act))
    out.write(np.ascontiguousarray(w_in, "<f4").tobytes())
    out.write(np.ascontiguousarray(w_rec, "<f4").tobytes())
    out.write(np.ascontiguousarray(np.asarray(w_out).T, "<f4").tobytes())  # H x V on disk
    out.write(_u64(len(vocab_words)))
    for w in vocab_words:
        out.write(_str(w))
    return out.getvalue()


def read_params(data_or_reader):
    """rnn.hpp:287-308 -> ((w_in, w_rec, w_out), act, vocab_words)."""
    r = data_or_reader if isinstance(data_or_reader, Reader) else Reader(data_or_reader)
    r.magic("RNLM", "rnn checkpoint")
    ver = r.u32()
    if ver != RNN_FORMAT_VERSION:
        raise DataError(f"rnn checkpoint: unsupported version {ver}")
    V, H = r.u64(), r.u64()
    if V < 1 or H < 1 or V > (1 << 26) or H > (1 << 20):
        raise DataError("rnn checkpoint: implausible dimensions")
    act = r.u8()
    w_in = r.f32s(V * H).reshape(V, H)
    w_rec = r.f32s(H * H).reshape(H, H)
    w_out = np.ascontiguousarray(r.f32s(H * V).reshape(H, V).T)
    n = r.u64()
    if n != V:
        raise DataError("rnn checkpoint: vocabulary size mismatch")
    words = [r.string() for _ in range(n)]
    return (w_in, w_rec, w_out), act, words


# ------------------------------------------------------------------ ROPT
def write_rmsprop(V, H, rho, eps, state) -> bytes:
    """rmsprop.hpp:139-149."""
    m_rec, m_in, m_out = state
    return (b"ROPT" + _u32(RMSPROP_FORMAT_VERSION) + _u64(V) + _u64(H) + _f64(rho) +
            _f64(eps) + np.ascontiguousarray(m_rec, "<f4").tobytes() +
            np.ascontiguousarray(m_in, "<f4").tobytes() +
            np.ascontiguousarray(m_out, "<f4").tobytes())


def read_rmsprop(data_or_reader):
    """rmsprop.hpp:151-166 -> (V, H, rho, eps, (m_rec, m_in, m_out))."""
    r = data_or_reader if isinstance(data_or_reader, Reader) else Reader(data_or_reader)
    r.magic("ROPT", "rmsprop state")
    ver = r.u32()
    if ver != RMSPROP_FORMAT_VERSION:
        raise DataError(f"rmsprop state: unsupported version {ver}")
    V, H = r.u64(), r.u64()
    rho, eps = r.f64(), r.f64()
    if not (0.0 < rho < 1.0):
        raise ValueError("rmsprop: rho must be in (0,1)")
    if not eps > 0.0:
        raise ValueError("rmsprop: eps must be > 0")
    m_rec = r.f32s(H * H).reshape(H, H)
    m_in = r.f32s(V)
    m_out = r.f32s(V)
    return V, H, rho, eps, (m_rec, m_in, m_out)


# ------------------------------------------------------------ RNBL / RBOP
BOTTLENECK_FORMAT_VERSION = 1


def write_bottleneck(params, vocab_words, act: int = 0) -> bytes:
    """write_bottleneck (compress.hpp:315-328): e, u, w_rec, d row-major."""
    e, u, w_rec, d = params
    V, P = e.shape
    H = w_rec.shape[0]
    out = io.BytesIO()
    out.write(b"RNBL" + _u32(BOTTLENECK_FORMAT_VERSION) + _u64(V) + _u64(H) + _u64(P) + _u8(act))
    for m in (e, u, w_rec, d):
        out.write(np.ascontiguousarray(m, "<f4").tobytes())
    out.write(_u64(len(vocab_words)))
    for w in vocab_words:
        out.write(_str(w))
    return out.getvalue()


def read_bottleneck(data_or_reader):
    """read_bottleneck (compress.hpp:330-354) -> ((e, u, w_rec, d), act, words)."""
    r = data_or_reader if isinstance(data_or_reader, Reader) else Reader(data_or_reader)
    r.magic("RNBL", "bottleneck checkpoint")
    ver = r.u32()
    if ver != BOTTLENECK_FORMAT_VERSION:
        raise DataError(f"bottleneck checkpoint: unsupported version {ver}")
    V, H, P = r.u64(), r.u64(), r.u64()
    if V < 1 or H < 1 or P < 1 or V > (1 << 26) or H > (1 << 20) or P > (1 << 20):
        raise DataError("bottleneck checkpoint: implausible dimensions")
    act = r.u8()
    if P > H:
        raise ValueError("BottleneckParams: P must not exceed H")
    e = r.f32s(V * P).reshape(V, P)
    u = r.f32s(P * H).reshape(P, H)
    w_rec = r.f32s(H * H).reshape(H, H)
    d = r.f32s(H * P).reshape(H, P)
    n = r.u64()
    if n != V:
        raise DataError("bottleneck checkpoint: vocabulary size mismatch")
    words = [r.string() for _ in range(n)]
    return (e, u, w_rec, d), act, words


def write_bottleneck_opt(V, H, P, rho, eps, state) -> bytes:
    """write_bottleneck_opt (compress.hpp:356-368): m_e, m_u, m_rec, m_d."""
    m_e, m_u, m_rec, m_d = state
    return (b"RBOP" + _u32(BOTTLENECK_FORMAT_VERSION) + _u64(V) + _u64(H) + _u64(P) + _f64(rho) +
            _f64(eps) + b"".join(np.ascontiguousarray(m, "<f4").tobytes()
                                 for m in (m_e, m_u, m_rec, m_d)))


def read_bottleneck_opt(data_or_reader):
    """read_bottleneck_opt (compress.hpp:370-386) -> (V, H, P, rho, eps, state)."""
    r = data_or_reader if isinstance(data_or_reader, Reader) else Reader(data_or_reader)
    r.magic("RBOP", "bottleneck optimizer state")
    ver = r.u32()
    if ver != BOTTLENECK_FORMAT_VERSION:
        raise DataError(f"bottleneck optimizer state: unsupported version {ver}")
    V, H, P = r.u64(), r.u64(), r.u64()
    rho, eps = r.f64(), r.f64()
    if V < 1 or H < 1 or P < 1:
        raise ValueError("opt state: V,H,P >= 1")
    if not (0.0 < rho < 1.0):
        raise ValueError("opt state: rho must be in (0, 1)")
    if not eps > 0.0:
        raise ValueError("opt state: eps must be > 0")
    m_e = r.f32s(V)
    m_u = r.f32s(P * H).reshape(P, H)
    m_rec = r.f32s(H * H).reshape(H, H)
    m_d = r.f32s(H * P).reshape(H, P)
    return V, H, P, rho, eps, (m_e, m_u, m_rec, m_d)


# ------------------------------------------------------------------ RNQZ
QUANTIZED_FORMAT_VERSION = 1


@dataclass
class QuantizedMatrix:
    """QuantizedMatrix (compress.hpp:423-448): per-matrix linear codes,
    packed without padding, least-significant bit first."""
    rows: int
    cols: int
    bits: int
    min: float
    max: float
    codes: bytes

    def step(self) -> float:
        rng = float(np.float32(self.max)) - float(np.float32(self.min))
        return rng / float((1 << self.bits) - 1) if rng > 0.0 else 0.0

    def code_array(self) -> np.ndarray:
        n = self.rows * self.cols
        b = np.unpackbits(np.frombuffer(self.codes, np.uint8), bitorder="little")
        b = b[: n * self.bits].reshape(n, self.bits).astype(np.uint32)
        return (b << np.arange(self.bits, dtype=np.uint32)).sum(axis=1, dtype=np.uint32)


def quantize_matrix(m, bits: int) -> QuantizedMatrix:
    """quantize_matrix (compress.hpp:450-479): step = (max - min) / (2^bits - 1),
    code = clamp(llround((x - min) / step)) in double."""
    if bits < 1 or bits > 16:
        raise ValueError("quantize: bits must be in [1, 16]")
    a = np.ascontiguousarray(m, np.float32)
    if a.size == 0:
        raise ValueError("quantize: empty matrix")
    mn, mx = np.float32(a.min()), np.float32(a.max())
    q = QuantizedMatrix(a.shape[0], a.shape[1] if a.ndim > 1 else 1, bits, float(mn), float(mx),
                        b"")
    n = a.size
    step = q.step()
    codes = np.zeros(n, np.int64)
    if step > 0.0:
        x = (a.ravel().astype(np.float64) - float(mn)) / step
        codes = np.clip(np.floor(x + 0.5), 0, (1 << bits) - 1).astype(np.int64)  # x >= 0: llround
    bitsarr = ((codes[:, None] >> np.arange(bits)) & 1).astype(np.uint8).ravel()
    q.codes = np.packbits(bitsarr, bitorder="little").tobytes()
    return q


def dequantize_matrix(q: QuantizedMatrix) -> np.ndarray:
    """dequantize_matrix (compress.hpp:481-488): float(min + step * code)."""
    v = float(np.float32(q.min)) + q.step() * q.code_array().astype(np.float64)
    return v.astype(np.float32).reshape(q.rows, q.cols)


@dataclass
class QuantizedModel:
    v: int
    h: int
    p: int
    act: int
    bits: int
    mats: tuple  # (e, u, w_rec, d) QuantizedMatrix
    words: list


def quantize_model(params, vocab_words, bits: int, act: int = 0) -> QuantizedModel:
    """quantize_model (compress.hpp:498-512)."""
    e, u, w_rec, d = params
    V, P = np.asarray(e).shape
    H = np.asarray(w_rec).shape[0]
    return QuantizedModel(V, H, P, act, bits, tuple(quantize_matrix(m, bits)
                                                    for m in (e, u, w_rec, d)),
                          list(vocab_words))


def dequantize_model(q: QuantizedModel):
    """dequantize_model (compress.hpp:514-523) -> ((e, u, w_rec, d), act, words)."""
    return tuple(dequantize_matrix(m) for m in q.mats), q.act, q.words


def write_quantized(q: QuantizedModel) -> bytes:
    """write_quantized (compress.hpp:575-586): RNQZ header, vocabulary, then
    each matrix's bits, min, max and code payload."""
    out = io.BytesIO()
    out.write(b"RNQZ" + _u32(QUANTIZED_FORMAT_VERSION) + _u64(q.v) + _u64(q.h) + _u64(q.p) +
              _u8(q.act) + _u64(len(q.words)))
    for w in q.words:
        out.write(_str(w))
    for m in q.mats:
        out.write(_u32(m.bits) + struct.pack("<f", m.min) + struct.pack("<f", m.max) + m.codes)
    return out.getvalue()


def quantized_size_bytes(q: QuantizedModel) -> int:
    """quantized_size_bytes (compress.hpp:563-573)."""
    n = 4 + 4 + 8 + 8 + 8 + 1 + 8 + sum(8 + len(w.encode()) for w in q.words)
    return n + sum(12 + len(m.codes) for m in q.mats)


def read_quantized(data_or_reader) -> QuantizedModel:
    """read_quantized (compress.hpp:588-617)."""
    r = data_or_reader if isinstance(data_or_reader, Reader) else Reader(data_or_reader)
    r.magic("RNQZ", "quantized model")
    ver = r.u32()
    if ver != QUANTIZED_FORMAT_VERSION:
        raise DataError(f"quantized model: unsupported version {ver}")
    V, H, P = r.u64(), r.u64(), r.u64()
    if V < 1 or H < 1 or P < 1 or P > H or V > (1 << 26) or H > (1 << 20):
        raise DataError("quantized model: implausible dimensions")
    act = r.u8()
    n = r.u64()
    if n != V:
        raise DataError("quantized model: vocabulary size mismatch")
    words = [r.string() for _ in range(n)]
    mats = []
    for rows, cols in ((V, P), (P, H), (H, H), (H, P)):
        bits = r.u32()
        if bits < 1 or bits > 16:
            raise DataError("quantized model: bits out of range")
        mn = struct.unpack("<f", r.take(4))[0]
        mx = struct.unpack("<f", r.take(4))[0]
        nbytes = (rows * cols * bits + 7) // 8
        try:
            codes = r.take(nbytes)
        except DataError:
            raise DataError("quantized model: truncated payload")
        mats.append(QuantizedMatrix(rows, cols, bits, mn, mx, codes))
    return QuantizedModel(V, H, P, act, mats[0].bits, tuple(mats), words)


# ---------------------------------------------------------- mt19937_64 text
def mt19937_64_text(seed: int) -> str:
    """`os << std::mt19937_64(seed)` as libstdc++ prints it: the 312 state
    words then the position index (312 right after seeding)."""
    M = (1 << 64) - 1
    x = [seed & M]
    for i in range(1, 312):
        x.append((6364136223846793005 * (x[-1] ^ (x[-1] >> 62)) + i) & M)
    return " ".join(str(v) for v in x) + " 312"


# ------------------------------------------------------------------ RTRN
CONFIG_ECHO = (  # trainer.hpp:412-432 (name, kind)
    ("nstate", "u64"), ("nproj", "u64"), ("noffset", "u32"), ("minibatch", "u32"),
    ("unroll", "u32"), ("eta", "f64"), ("rho", "f64"), ("eps", "f64"), ("clip", "f64"),
    ("mode", "u8"), ("nce_k", "u32"), ("noise_floor", "f64"), ("max_epochs", "u32"),
    ("seed", "u64"), ("act", "u8"), ("divergence_factor", "f64"), ("valid_limit", "u64"),
    ("valid_shards", "u32"), ("init_range", "f64"),
)


def write_config_echo(cfg) -> bytes:
    pk = {"u64": _u64, "u32": _u32, "u8": _u8, "f64": _f64}
    return b"".join(pk[k](getattr(cfg, n) if k == "f64" else int(getattr(cfg, n)))
                    for n, k in CONFIG_ECHO)


def check_config_echo(r: Reader, cfg):
    rd = {"u64": r.u64, "u32": r.u32, "u8": r.u8, "f64": r.f64}
    ok = True
    for n, k in CONFIG_ECHO:
        v = rd[k]()
        if n == "max_epochs":  # only a stopping rule; a resumed run may raise it
            continue
        want = getattr(cfg, n)
        ok = ok and (v == (want if k == "f64" else int(want)))
    if not ok:
        raise DataError("trainer checkpoint: configuration does not match this run")


def write_trainer(cfg, epoch, eta, best, bad, initial, rng_text, cursors, hidden, params,
                  vocab_words, opt_state, model: str = "rnn") -> bytes:
    """trainer.hpp:274-292.  model: "rnn" (Traits = StandardTraits: RNLM +
    ROPT) or "bottleneck" (BottleneckTraits: RNBL + RBOP, compress.hpp:404-414)."""
    out = io.BytesIO()
    out.write(b"RTRN" + _u32(TRAINER_FORMAT_VERSION) + write_config_echo(cfg))
    out.write(_u32(epoch) + _f64(eta) + _f64(best) + _u32(bad) + _f64(initial))
    out.write(_str(rng_text))
    out.write(_u64(len(cursors)))
    out.write(np.ascontiguousarray(cursors, "<u8").tobytes())
    out.write(np.ascontiguousarray(hidden, "<f4").tobytes())
    if model == "bottleneck":
        V, P = params[0].shape
        H = params[2].shape[0]
        out.write(write_bottleneck(params, vocab_words, cfg.act))
        out.write(write_bottleneck_opt(V, H, P, cfg.rho, cfg.eps, opt_state))
    else:
        V, H = params[0].shape
        out.write(write_params(params, vocab_words, cfg.act))
        out.write(write_rmsprop(V, H, cfg.rho, cfg.eps, opt_state))
    out.write(b"TEND")
    return out.getvalue()


def read_trainer(data: bytes, cfg, n_streams: int, hidden_size: int, L: int,
                 model: str = "rnn"):
    """trainer.hpp:300-336; returns a dict of the restored state."""
    r = Reader(data)
    r.magic("RTRN", "trainer checkpoint")
    ver = r.u32()
    if ver != TRAINER_FORMAT_VERSION:
        raise DataError(f"trainer checkpoint: unsupported version {ver}")
    check_config_echo(r, cfg)
    st = dict(epoch=r.u32(), eta=r.f64(), best=r.f64(), bad=r.u32(), initial=r.f64())
    st["rng_text"] = r.string()
    n = r.u64()
    if n != n_streams:
        raise DataError("trainer checkpoint: cursor count mismatch")
    cur = np.frombuffer(r.take(8 * n), dtype="<u8").astype(np.int64)
    if np.any(cur < 0) or np.any(cur >= L):
        raise DataError("trainer checkpoint: cursor out of range")
    st["cursors"] = cur
    st["hidden"] = r.f32s(n * hidden_size).reshape(n, hidden_size)
    if model == "bottleneck":
        st["params"], st["act"], st["vocab"] = read_bottleneck(r)
        st["opt"] = read_bottleneck_opt(r)[5]
    else:
        st["params"], st["act"], st["vocab"] = read_params(r)
        _, _, _, _, st["opt"] = read_rmsprop(r)
    r.magic("TEND", "trainer checkpoint trailer")
    return st
