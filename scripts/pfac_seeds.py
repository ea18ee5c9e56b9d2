"""Diagnostics: the bigram-chain PPL match (tests/test_gpu_bf16.py) over
several init seeds -- reference (oracle) vs the bf16 trainer with the
in-place softmax (DL_PFAC=0) and the shifted-exponential softmax (DL_PFAC=1)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1502_00512_b200 as dl

orc = oracle.Orc()
V, H = int(os.environ.get("V", 2000)), int(os.environ.get("H", 128))
rng = np.random.default_rng(555)
succ = rng.integers(3, V, (V, 4))
ids = [1]
w = 3
while len(ids) < 28100:
    if rng.random() < 0.1:
        ids += [2, 1]
        w = int(rng.integers(3, V))
    else:
        w = int(succ[w, rng.integers(0, 4)])
    ids.append(w)
ids = np.array(ids, np.uint32)
tr, va = ids[:24000], ids[24000:28000]
kw = dict(nstate=H, noffset=16, minibatch=8, unroll=8, eta=0.05, max_epochs=1, mode=1)
res = {"0": [], "1": [], "fp32": []}
for seed in range(int(os.environ.get("SEED0", 1)), int(os.environ.get("SEED0", 1)) + int(os.environ.get("SEEDS", 8))):
    params0 = orc.init_uniform(V, H, seed)
    ref = orc.train(oracle.TrainConfig(**kw), params0, tr, va)["logs"][0][2]
    row = []
    for pf in ("0", "1", "fp32"):
        os.environ["DL_PFAC"] = "1" if pf == "fp32" else pf
        t = dl.Trainer(dl.TrainConfig(**kw), [p.copy() for p in params0], dl.make_vocab(V), tr,
                       va, "fp32" if pf == "fp32" else "bf16")
        try:
            t.train()
            d = t.logs[0].valid_ppl / ref - 1
        except dl.DataError as e:
            print("seed", seed, pf, "failed:", e, flush=True)
            d = float("nan")
        res[pf].append(d)
        row.append(f"{100 * d:+.2f}%")
        t.model.close()
    print("seed", seed, "ref", f"{ref:.2f}", "pfac0/pfac1/fp32", " ".join(row), flush=True)
for k, v in res.items():
    v = np.array(v)
    v = v[np.isfinite(v)]
    print(k, f"mean {100 * v.mean():+.2f}%  std {100 * v.std():.2f}%  max|.| {100 * np.abs(v).max():.2f}%")
