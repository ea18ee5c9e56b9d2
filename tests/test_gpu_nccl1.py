"""The NCCL code paths on one GPU: a real
one-rank NcclComm (comm.cu) drives the data-parallel window -- dW_out /
dW_rec allreduce before clip, the gathered (ids, dpre) W_in rows, the loss
allreduce -- and the data-parallel + vocabulary-parallel output layer
(hidden-state allgather, block log-sum-exp exchange, dh reduce-scatter, the
fused dW_out + rmsprop epilogue under a communicator); each must train like
a context without a communicator (identity exchanges)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# libdesklm_cuda.so binds libnccl.so.2 by soname: loaded after torch it
# uses torch's NCCL (2.28), as bench.py's multi-GPU runs do (torch.distributed
# is up first)
import torch  # noqa: E402,F401


def _train(dl, params, ids, V, H, precision, mode, windows=12):
    m = dl.GpuRnn(V, H, 0, precision)
    if mode is not None:
        m.comm_init(dl.comm_unique_id(), 1, 0)
        if mode == "dp":
            m.set_vocab_shard("dp")
    m.set_params(*params)
    m.set_opt(None, None, None, 0.9995, 1e-6)
    m.trainer_init(ids, 2, 128, 4, 1.0)
    l1, sk = m.trainer_run(0, windows, 0.01)
    out = (l1, sk, m.params(), m.opt(), m.trainer_state())
    m.close()
    return out


def _setup(orc):
    V, H = 4096, 256
    ids = orc.random_stream(71, V, 40000)[:40000]
    rng = np.random.default_rng(5)
    params = tuple(rng.uniform(-0.1, 0.1, s).astype(np.float32) for s in ((V, H), (H, H), (V, H)))
    return V, H, ids, params


@pytest.mark.parametrize("precision,mode", [("fp32", "dense"), ("fp32", "dp"),
                                            ("bf16", "dense"), ("bf16", "dp")])
def test_one_rank_nccl_matches_single_context(orc, monkeypatch, precision, mode):
    import paper_1502_00512_b200 as dl
    V, H, ids, params = _setup(orc)
    if precision == "bf16" and mode == "dense":
        # dense DP sums a bf16 dW_out: the single context's matching path is
        # the unfused bf16 gradient + row sums (env read at context creation)
        for k in ("DL_FUSE_OUT", "DL_FORK_OUT", "DL_FORK_LATE"):
            monkeypatch.setenv(k, "0")
    ref = _train(dl, params, ids, V, H, precision, None)
    monkeypatch.delenv("DL_FUSE_OUT", raising=False)
    monkeypatch.delenv("DL_FORK_OUT", raising=False)
    monkeypatch.delenv("DL_FORK_LATE", raising=False)
    got = _train(dl, params, ids, V, H, precision, mode)
    assert got[1] == ref[1] == 0
    # fp32: identity exchanges, the same sums (the gathered W_in rows and the
    # block log-sum-exp combine reorder nothing); bf16 dense DP sums dW_out in
    # bf16 before the update (the single context fuses it in fp32)
    rel = 1e-9 if precision == "fp32" else 1e-3
    assert got[0] == pytest.approx(ref[0], rel=rel)
    for a, b in zip(got[2] + got[3], ref[2] + ref[3]):
        scale = max(float(np.abs(b).max()), 1e-30)
        if precision == "fp32":
            assert float(np.abs(a - b).max()) <= 1e-6 * scale
        else:
            # (rmsprop's early steps, ~eta / sqrt(1 - rho) per element, follow
            # the sign of tiny gradients: the bf16-rounded sum flips a few)
            rel = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
            assert rel <= 1e-2, rel
    assert np.array_equal(got[4][0], ref[4][0])  # cursors: the same schedule


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_dense_dp_chunked_allreduce_is_exact(orc, monkeypatch, precision):
    """The dense-DP dW_out GEMM + allreduce in V chunks (the allreduce of
    chunk i under the GEMM of chunk i+1) gives the unchunked result bit for
    bit: every element is the same dot product and the same rank sum."""
    import paper_1502_00512_b200 as dl
    V, H, ids, params = _setup(orc)
    monkeypatch.setenv("DL_DP_CHUNKS", "1")
    one = _train(dl, params, ids, V, H, precision, "dense", windows=6)
    monkeypatch.setenv("DL_DP_CHUNKS", "5")
    five = _train(dl, params, ids, V, H, precision, "dense", windows=6)
    assert one[0] == five[0]
    for a, b in zip(one[2] + one[3], five[2] + five[3]):
        assert np.array_equal(a, b)


def test_one_rank_nccl_scoring_and_window(orc):
    """Scoring and a single window through the one-rank communicator with the
    vocabulary-sharded output layer (block lse exchange) in fp32."""
    import paper_1502_00512_b200 as dl
    V, H, T, B = 2000, 64, 6, 8
    params = orc.init_uniform(V, H, 13)
    ids = orc.random_stream(3, V, 3000)
    m = dl.GpuRnn(V, H, 0, "fp32")
    m.comm_init(dl.comm_unique_id(), 1, 0)
    m.set_vocab_shard(True)
    m.set_params(*params)
    want = orc.sharded_ppl(params, 0, ids, 8)
    got = dl.sharded_perplexity(m, ids, 8)
    assert got.predicted == want["predicted"]
    assert got.total_logprob == pytest.approx(want["total_logprob"], rel=1e-5)
    rng = np.random.default_rng(1)
    x = rng.integers(0, V, (T, B)).astype(np.uint32)
    y = rng.integers(2, V, (T, B)).astype(np.uint32)
    w = np.ones((T, B), np.uint8)
    h0 = np.full((B, H), 0.5, np.float32)
    ref = orc.bptt(params, 0, x, y, w, h0, 1.0 / (T * B), 1.0)
    res, hf = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, 1.0 / (T * B), 1.0)
    assert res.loss == pytest.approx(ref["loss"], rel=1e-5)
    g_in, g_rec, g_out = m.grads()
    for a, b in ((g_in, ref["g_in_dense"]), (g_rec, ref["g_rec"]), (g_out, ref["g_out"])):
        assert float(np.abs(a - b).max()) <= 1e-4 * float(np.abs(b).max()) + 1e-9
