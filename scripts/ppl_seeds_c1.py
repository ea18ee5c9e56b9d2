"""Diagnostics: the PPL match over the init seeds of a fixture (default
tests/golden/ppl_match_c1.npz, seed 1) and its <name>_seeds.npz, per
precision: device valid ppl vs the reference trainer's, per seed.
  python scripts/ppl_seeds_c1.py bf16,fp32 [ppl_match_h1024]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1502_00512_b200 as dl
GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
FX = sys.argv[2] if len(sys.argv) > 2 else "ppl_match_c1"
g = np.load(os.path.join(GOLD, FX + ".npz"))
s = np.load(os.path.join(GOLD, FX + "_seeds.npz"))
V, H = int(g["V"]), int(g["H"])
seeds = [1] + [int(x) for x in s["seeds"]]
refs = [float(g["logs"][0][2])] + [float(l[2]) for l in s["logs"]]
for prec in (sys.argv[1].split(",") if len(sys.argv) > 1 else ("bf16", "fp32")):
    d = []
    for seed, ref in zip(seeds, refs):
        cfg = dl.TrainConfig(nstate=H, noffset=128, minibatch=8, unroll=8, eta=float(g["eta"]),
                             max_epochs=1, mode=1)
        t = dl.Trainer(cfg, dl.init_uniform(V, H, seed), dl.make_vocab(V), g["train"], g["valid"],
                       prec)
        t.train()
        d.append(t.logs[0].valid_ppl / ref - 1)
        t.model.close()
    d = np.array(d)
    print(FX, prec, " ".join(f"{100 * v:+.2f}%" for v in d), f"| mean {100 * d.mean():+.2f}%", flush=True)
