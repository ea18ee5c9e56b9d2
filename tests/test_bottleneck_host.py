"""Host side of the bottleneck model (no GPU): parameter count, the
bit-exact mt19937_64 init and the RNBL / RBOP byte layouts against the
reference's own fixtures (tests/golden/bn_*.npz, made by oracle/_ref)."""
import glob
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_param_count_matches_reference_formula():
    from paper_1502_00512_b200.bottleneck import bottleneck_param_count
    assert bottleneck_param_count(10000, 128, 32) == 10000 * 32 + 32 * 128 + 128 * 128 + 128 * 32
    with pytest.raises(ValueError):
        bottleneck_param_count(0, 4, 2)


def test_init_uniform_matches_oracle(orc):
    from paper_1502_00512_b200.bottleneck import bn_init_uniform
    for V, H, P, seed in ((50, 16, 8, 7), (300, 32, 32, 11)):
        got = bn_init_uniform(V, H, P, seed)
        want = orc.bn_init_uniform(V, H, P, seed)
        for a, b in zip(got, want):
            assert np.array_equal(a, b)
    with pytest.raises(ValueError):
        bn_init_uniform(10, 4, 8, 1)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "bn_[0-9]*.npz"))))
def test_rnbl_rbop_bytes_match_reference(path):
    from paper_1502_00512_b200 import formats, make_vocab
    g = np.load(path)
    params = (g["e"], g["u"], g["w_rec"], g["d"])
    V, H, P = int(g["V"]), int(g["H"]), int(g["P"])
    rnbl = formats.write_bottleneck(params, make_vocab(V), int(g["act"]))
    assert rnbl == g["rnbl"].tobytes()
    state = (g["m_e"], g["m_u"], g["m_rec"], g["m_d"])
    rbop = formats.write_bottleneck_opt(V, H, P, 0.9995, 1e-6, state)
    assert rbop == g["rbop"].tobytes()
    (e, u, w_rec, d), act, words = formats.read_bottleneck(rnbl)
    assert act == int(g["act"]) and words == make_vocab(V)
    for a, b in zip((e, u, w_rec, d), params):
        assert np.array_equal(a, b)
    V2, H2, P2, rho, eps, st = formats.read_bottleneck_opt(rbop)
    assert (V2, H2, P2, rho, eps) == (V, H, P, 0.9995, 1e-6)
    for a, b in zip(st, state):
        assert np.array_equal(a, b)
    with pytest.raises(formats.DataError):
        formats.read_bottleneck(b"RNLM" + rnbl[4:])


@pytest.mark.parametrize("bits", [3, 8, 13])
def test_rnqz_bytes_and_dequantization_match_reference(bits):
    """quantize_model / write_quantized / read_quantized / dequantize_model
    (compress.hpp:417-617) against the reference's bytes and values."""
    from paper_1502_00512_b200 import formats, make_vocab
    g = np.load(os.path.join(GOLD, "rnqz.npz"))
    params = (g["e"], g["u"], g["w_rec"], g["d"])
    q = formats.quantize_model(params, make_vocab(params[0].shape[0]), bits, act=1)
    blob = formats.write_quantized(q)
    assert blob == g[f"rnqz_{bits}"].tobytes()
    assert formats.quantized_size_bytes(q) == len(blob)
    q2 = formats.read_quantized(blob)
    dq, act, words = formats.dequantize_model(q2)
    assert act == 1 and words == make_vocab(params[0].shape[0])
    for a, k in zip(dq, ("e", "u", "w_rec", "d")):
        assert np.array_equal(a, g[f"dq_{bits}_{k}"]), k
    with pytest.raises(formats.DataError):
        formats.read_quantized(blob[:-3])
