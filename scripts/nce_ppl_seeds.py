"""Diagnostics: NCE training (LossMode::kNce, the reference's default) on the
C1 PPL-match fixture's streams, one epoch per init seed, bf16 vs fp32 (the
fp32 trainer is pinned to the oracle's epochs in tests/test_gpu_nce.py):
validation perplexity per seed and the seed-mean difference.
  python scripts/nce_ppl_seeds.py [n_seeds] [fixture] [eta]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1502_00512_b200 as dl
GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
FX = sys.argv[2] if len(sys.argv) > 2 else "ppl_match_c1"
ETA = float(sys.argv[3]) if len(sys.argv) > 3 else 2e-3
g = np.load(os.path.join(GOLD, FX + ".npz"))
V, H = int(g["V"]), int(g["H"])
res = {}
for prec in ("fp32", "bf16"):
    ppl = []
    for seed in range(1, n + 1):
        cfg = dl.TrainConfig(nstate=H, noffset=128, minibatch=8, unroll=8, eta=ETA,
                             max_epochs=1, mode=0, seed=seed, divergence_factor=1e30)
        t = dl.Trainer(cfg, dl.init_uniform(V, H, seed), dl.make_vocab(V), g["train"], g["valid"],
                       prec)
        t.train()
        ppl.append(t.logs[0].valid_ppl)
        t.model.close()
    res[prec] = np.array(ppl)
    print(FX, "NCE", prec, " ".join(f"{p:.2f}" for p in ppl), flush=True)
d = res["bf16"] / res["fp32"] - 1
print("bf16 vs fp32 per seed:", " ".join(f"{100 * v:+.2f}%" for v in d),
      f"| seed mean {100 * (res['bf16'].mean() / res['fp32'].mean() - 1):+.2f}%")
