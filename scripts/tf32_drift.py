"""Diagnostics: C1 one-epoch training in fp32 mode with 3xTF32 vs SIMT GEMMs;
the trained parameters re-scored by both engines."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
g = np.load(os.path.join(GOLD, "ppl_match_c1.npz"))
V, H = int(g["V"]), int(g["H"])
res = {}
import paper_1502_00512_b200 as dl
for simt, prec in (("0", "tf32x3"), ("1", "fp32")):
    params = dl.init_uniform(V, H, int(g["init_seed"]))
    cfg = dl.TrainConfig(nstate=H, noffset=128, minibatch=8, unroll=8, eta=float(g["eta"]),
                         max_epochs=1, mode=1)
    t = dl.Trainer(cfg, params, dl.make_vocab(V), g["train"], g["valid"], prec)
    t.train()
    res[simt] = t.params()
    print("DL_SIMT", simt, "initial", t.initial_ppl, "epoch1", t.logs[0].valid_ppl, t.logs[0].train_loss,
          "ref", float(g["logs"][0][2]), flush=True)
for simt, prec in (("0", "tf32x3"), ("1", "fp32")):
    for trained in ("0", "1"):
        m = dl.GpuRnn(V, H, 0, prec)
        m.set_params(*res[trained])
        print(f"score engine simt={simt} params from simt={trained}:",
              dl.sharded_perplexity(m, g["valid"], 8).perplexity, flush=True)
        m.close()
a, b = res["0"], res["1"]
for x, y, n in zip(a, b, ("w_in", "w_rec", "w_out")):
    print(n, "max abs diff", float(np.abs(x - y).max()), "rel", float(np.abs(x - y).max() / np.abs(y).max()))
