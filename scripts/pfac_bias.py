"""Diagnostics: gradient error and scale bias of the bf16 output layer in a
TRAINED state.  Trains the C1 model (ppl_match_c1 corpus, seed 2) in the fp32
device mode for N windows, then scores one window of the corpus with the C
oracle (fp32 with double accumulation, backprop.hpp) and with the bf16 mode
under the shifted-exponential softmax (DL_PFAC=1) and the in-place kernel
(DL_PFAC=0): per gradient, rel-L2 error and beta = <got, ref> / <ref, ref> - 1
(a systematic scale bias)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_1502_00512_b200 as dl

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
g = np.load(os.path.join(GOLD, "ppl_match_c1.npz"))
V, H = int(g["V"]), int(g["H"])
nwin = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 2
orc = oracle.Orc()
cfg = dl.TrainConfig(nstate=H, noffset=128, minibatch=8, unroll=8, eta=0.05, max_epochs=1, mode=1)
tr = g["train"][: nwin * 8 * 8 + 1]
t = dl.Trainer(cfg, dl.init_uniform(V, H, seed), dl.make_vocab(V), tr, g["valid"][:1000], "fp32")
t.train()
params = t.params()
t.model.close()
T, B = 8, 64
rng = np.random.default_rng(1)
for trial in range(3):
    s0 = int(rng.integers(0, len(g["valid"]) - T * B - 2))
    ids = g["valid"][s0:s0 + T * B + 1]
    x = ids[:-1].reshape(T, B).astype(np.uint32)
    y = ids[1:].reshape(T, B).astype(np.uint32)
    w = (y != 1).astype(np.uint8)
    h0 = rng.uniform(0, 1, (B, H)).astype(np.float32)
    scale = 1.0 / (T * B)
    want = orc.bptt(params, 0, x, y, w, h0, scale, 1e9)
    line = [f"trial {trial} loss {want['loss']:.4f}"]
    for pf in ("1", "0"):
        os.environ["DL_PFAC"] = pf
        os.environ["DL_G16"] = "0"
        m = dl.GpuRnn(V, H, 0, "bf16")
        m.set_params(*params)
        r, hf = dl.bptt_run(m, dl.WindowBatch(x, y, w), h0, scale, 1e9)
        gi, gr, go = m.grads()
        m.close()
        for name, got, ref in (("g_out", go, want["g_out"]), ("g_rec", gr, want["g_rec"]),
                               ("g_in", gi, want["g_in_dense"])):
            got = got.astype(np.float64); ref = ref.astype(np.float64)
            err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            beta = float(np.dot(got.ravel(), ref.ravel()) / np.dot(ref.ravel(), ref.ravel()) - 1)
            line.append(f"pfac{pf} {name} err {err:.2e} beta {beta:+.2e}")
        line.append(f"pfac{pf} loss {r.loss / want['loss'] - 1:+.2e}")
    print(" | ".join(line), flush=True)
