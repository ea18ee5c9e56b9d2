"""Multi-process (world_size 2, gloo, CPU) checks of the data-parallel
decomposition the B200 trainer uses:

* rank r owns global streams g*G*B + r*B + b of every group, so the union of
  the ranks' cursors is exactly the reference's floor(i*L/N) set for the
  global minibatch G*B (dl_rank_cursors, the C-ABI host function the
  device trainer calls);
* per-rank windows with loss_scale 1/(G*B*T), summed across ranks by an
  allreduce, reproduce the single-process window over all G*B streams
  (loss, W_rec and W_out gradients; W_in rows by word) -- the exchange the
  NCCL path performs before clip + rmsprop.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_1502_00512_b200 as dl
        orc = oracle.Orc()
        V, H, T, B, noffset = 40, 8, 5, 3, 2
        L = 300
        ids = orc.random_stream(5, V, L + 8)[:L]
        # ---- stream partition
        mine = dl.rank_cursors(L, noffset, B, world, rank)
        allc = [torch.zeros(len(mine), dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allc, torch.from_numpy(mine))
        if rank == 0:
            Bg = B * world
            N = noffset * Bg
            want = [i * L // N for i in range(N)]
            got = [None] * N
            for r in range(world):
                for g in range(noffset):
                    for b in range(B):
                        got[g * Bg + r * B + b] = int(allc[r][g * B + b])
            out["cursors_ok"] = got == want
        # ---- one window: global group 0 vs the rank-local slices
        Bg = B * world
        gcur = dl.rank_cursors(L, noffset, Bg, 1, 0)[:Bg]
        x, y, w = orc.window_build(ids, gcur, 0, Bg, T)
        params = orc.init_uniform(V, H, 3)
        h0 = np.random.default_rng(1).uniform(-0.5, 0.5, (Bg, H)).astype(np.float32)
        full = orc.bptt(params, 0, x, y, w, h0, 1.0 / (Bg * T), 3.4e38)
        sl = slice(rank * B, (rank + 1) * B)
        loc = orc.bptt(params, 0, np.ascontiguousarray(x[:, sl]), np.ascontiguousarray(y[:, sl]),
                       np.ascontiguousarray(w[:, sl]), np.ascontiguousarray(h0[sl]),
                       1.0 / (Bg * T), 3.4e38)
        t = {k: torch.from_numpy(np.ascontiguousarray(loc[k]).astype(np.float64))
             for k in ("g_rec", "g_out", "g_in_dense")}
        loss = torch.tensor([loc["loss"]], dtype=torch.float64)
        for v in list(t.values()) + [loss]:
            dist.all_reduce(v)
        if rank == 0:
            out["loss"] = (float(loss[0]), full["loss"])
            for k in t:
                ref = full[k].astype(np.float64)
                err = float(np.abs(t[k].numpy() - ref).max())
                out[k] = err / (np.abs(ref).max() + 1e-30)
            hf_ok = np.allclose(loc["h_final"], full["h_final"][sl], rtol=0, atol=0)
            out["hfinal_ok"] = bool(hf_ok)
    finally:
        dist.destroy_process_group()


def test_dp_decomposition_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out["cursors_ok"]
    a, b = out["loss"]
    assert a == pytest.approx(b, rel=1e-12)
    for k in ("g_rec", "g_out", "g_in_dense"):
        assert out[k] < 1e-5, (k, out[k])
    assert out["hfinal_ok"]


def _vshard_worker(rank, world, port, out):
    """The two vocabulary-parallel exchanges:
    per-row block log-sum-exps gathered from every rank and combined, the
    target logit summed from its owner, dS local to the shard, dh summed
    (vshard) or reduce-scattered over the gathered rows (dp + vocab-parallel
    output)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        M, V, H = 12, 50, 6
        h = rng.uniform(0, 1, (world * M, H))        # rank-blocked rows (dpv gathers them)
        w_out = rng.uniform(-1, 1, (V, H))
        y = rng.integers(0, V, world * M)
        scale = 1.0 / (world * M)
        # rank r owns rows [r V / G, (r+1) V / G) of W_out (dl_set_vocab_shard)
        v0, v1 = rank * V // world, (rank + 1) * V // world
        s = h @ w_out[v0:v1].T                        # local logits over all gathered rows
        mx = s.max(axis=1)
        blk = mx + np.log(np.exp(s - mx[:, None]).sum(axis=1))
        allb = [torch.zeros(world * M, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allb, torch.from_numpy(blk))
        B = np.stack([t.numpy() for t in allb])
        gm = B.max(axis=0)
        lse = gm + np.log(np.exp(B - gm).sum(axis=0))
        own = (y >= v0) & (y < v1)
        tl = torch.from_numpy(np.where(own, s[np.arange(world * M), np.clip(y - v0, 0, v1 - v0 - 1)], 0.0))
        dist.all_reduce(tl)
        loss = float((scale * (lse - tl.numpy())).sum())
        ds = scale * np.exp(s - lse[:, None])
        ds[np.arange(world * M)[own], (y - v0)[own]] -= scale
        dh_part = torch.from_numpy(ds @ w_out[v0:v1])
        # dp + vocab-parallel output: each rank keeps its own M rows of dh
        mine = torch.zeros(M, H, dtype=torch.float64)
        dist.reduce_scatter(mine, list(dh_part.reshape(world, M, H).unbind(0)))
        if rank == 0:
            full = h @ w_out.T
            fm = full.max(axis=1)
            flse = fm + np.log(np.exp(full - fm[:, None]).sum(axis=1))
            floss = float((scale * (flse - full[np.arange(world * M), y])).sum())
            fds = scale * np.exp(full - flse[:, None])
            fds[np.arange(world * M), y] -= scale
            fdh = fds @ w_out
            out["loss"] = (loss, floss)
            out["lse"] = float(np.abs(lse - flse).max())
            out["dh0"] = float(np.abs(mine.numpy() - fdh[:M]).max())
            out["dw_block"] = float(np.abs(ds.T @ h - (fds.T @ h)[v0:v1]).max())
    finally:
        dist.destroy_process_group()


def test_vocab_parallel_exchanges_gloo_world2():
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_vshard_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res["loss"][0] == pytest.approx(res["loss"][1], rel=1e-12)
    assert res["lse"] < 1e-12 and res["dh0"] < 1e-12 and res["dw_block"] < 1e-12
