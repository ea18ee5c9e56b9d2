"""Single-GPU checks of the multi-GPU code paths: the gathered-window W_in
gradient the data-parallel trainer computes after its NCCL allgather, and
the concurrent (side-stream) W_out update being bit-identical to the
sequential one."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_gathered_embed_follows_global_processing_order():
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200._lib import check, load
    G, T, B, V, H = 4, 3, 5, 20, 24
    rng = np.random.default_rng(9)
    x = rng.integers(0, V, (G, T, B)).astype(np.uint32)
    x[:, :, 0] = 1  # a frequent word, like bos
    d = rng.standard_normal((G, T, B, H)).astype(np.float32)
    clip = np.float32(1.5)
    want = np.zeros((V, H), np.float32)
    for t in range(T - 1, -1, -1):  # processing order: t desc, global stream asc
        for r in range(G):
            for b in range(B):
                want[x[r, t, b]] += np.float32(1.0) * d[r, t, b]
    touched = np.zeros(V, bool)
    touched[np.unique(x)] = True
    want[touched] = np.minimum(clip, np.maximum(-clip, want[touched]))
    m = dl.GpuRnn(V, H, 0, "fp32")
    got = np.empty((V, H), np.float32)
    check(load().dl_test_embed(m.handle, G, T, B, x.ctypes.data, d.ctypes.data, float(clip),
                               got.ctypes.data), m.handle)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("H", [100, 256, 2048])
def test_embed_rows_all_segment_lengths_bitexact(H):
    """W_in gradient rows for segments of every length class (kernels.cu):
    1-64 rows on the warp kernel (next row's loads in flight), 65-168 rows
    (one staged pass of k_embed_long) and ~500 rows (double-buffered
    passes): each word's rows summed in the reference's processing order,
    bit-exact; H = 100 takes the unaligned scalar paths."""
    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200._lib import check, load
    G, T, B, V = 1, 16, 64, 400
    rng = np.random.default_rng(H)
    x = rng.integers(20, V, (G, T, B)).astype(np.uint32)
    flat = x.reshape(-1)
    pos = rng.permutation(flat.size)
    flat[pos[:500]] = 1      # ~500-row segment
    flat[pos[500:600]] = 2   # 100 rows
    for k, n in enumerate((64, 65, 40, 9, 8)):
        off = 600 + sum((64, 65, 40, 9, 8)[:k])
        flat[pos[off:off + n]] = 3 + k
    d = rng.standard_normal((G, T, B, H)).astype(np.float32)
    clip = np.float32(40.0)
    want = np.zeros((V, H), np.float32)
    for t in range(T - 1, -1, -1):
        for b in range(B):
            want[x[0, t, b]] += d[0, t, b]
    touched = np.zeros(V, bool)
    touched[np.unique(x)] = True
    want[touched] = np.minimum(clip, np.maximum(-clip, want[touched]))
    m = dl.GpuRnn(V, H, 0, "fp32")
    got = np.empty((V, H), np.float32)
    check(load().dl_test_embed(m.handle, G, T, B, x.ctypes.data, d.ctypes.data, float(clip),
                               got.ctypes.data), m.handle)
    assert np.array_equal(got, want)


def test_concurrent_wout_update_is_bitexact(orc):
    import paper_1502_00512_b200 as dl
    V, H = 4096, 1024
    tr, va = orc.random_stream_pair(12, V, 40000, 2000)
    params = orc.init_uniform(V, H, 4)
    kw = dict(nstate=H, noffset=2, minibatch=128, unroll=8, eta=0.01, max_epochs=1, mode=1)
    res = []
    for flag in ("0", "1"):
        os.environ["DL_FORK_OUT"] = flag
        os.environ["DL_FUSE_OUT"] = "0"  # (the fused epilogue update takes precedence)
        try:
            t = dl.Trainer(dl.TrainConfig(**kw), params, dl.make_vocab(V), tr[:40000], va, "bf16")
        finally:
            os.environ.pop("DL_FORK_OUT", None)
            os.environ.pop("DL_FUSE_OUT", None)
        t.model.trainer_run(0, 5, 0.01)
        res.append((t.model.params(), t.model.opt()))
        t.model.close()
    for a, b in zip(res[0][0] + res[0][1], res[1][0] + res[1][1]):
        assert np.array_equal(a, b)
