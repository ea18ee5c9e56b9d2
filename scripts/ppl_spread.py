"""Diagnostics: spread of the C1 PPL-match result under 1-ulp perturbations of
one W_rec element (the chaotic sensitivity of one epoch at eta 0.05), per
precision mode; compare with tests/golden/ppl_match_c1.npz (reference)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1502_00512_b200 as dl
GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
fx = sys.argv[1] if len(sys.argv) > 1 else "ppl_match_c1.npz"
g = np.load(os.path.join(GOLD, fx))
V, H = int(g["V"]), int(g["H"])
ref, ref_loss = float(g["logs"][0][2]), float(g["logs"][0][1])
precs = sys.argv[2].split(",") if len(sys.argv) > 2 else ("fp32", "tf32x3", "bf16")
for prec in precs:
    vals, losses = [], []
    for k in range(-1, 4):
        params = [p.copy() for p in dl.init_uniform(V, H, int(g["init_seed"]))]
        if k >= 0:
            f = params[1].reshape(-1)
            f[k] = np.nextafter(f[k], np.float32(1))
        cfg = dl.TrainConfig(nstate=H, noffset=128, minibatch=8, unroll=8, eta=float(g["eta"]),
                             max_epochs=1, mode=1)
        t = dl.Trainer(cfg, params, dl.make_vocab(V), g["train"], g["valid"], prec)
        t.train()
        vals.append(t.logs[0].valid_ppl / ref - 1)
        losses.append(t.logs[0].train_loss / ref_loss - 1)
        t.model.close()
    print(prec, "valid ppl", " ".join(f"{100 * v:+.2f}%" for v in vals), "| train loss",
          " ".join(f"{100 * v:+.2f}%" for v in losses), flush=True)
