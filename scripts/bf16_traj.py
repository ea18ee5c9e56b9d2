"""Diagnostics: the per-window training-loss trajectory of one PPL-match epoch
(tests/golden/<fixture>) in fp32 and bf16, and whether the bf16 trainer's
reported window loss is the model's loss: at a few points the bf16-trained
parameters are copied into an fp32 context and the next window is scored by
both (no update)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1502_00512_b200 as dl
GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
fx = sys.argv[1] if len(sys.argv) > 1 else "ppl_match_h1024.npz"
g = np.load(os.path.join(GOLD, fx))
V, H = int(g["V"]), int(g["H"])
eta = float(g["eta"])
ids = np.ascontiguousarray(g["train"], np.uint32)
L = len(ids)
NOFF, B, T = 128, 8, 8
windows = ((L + NOFF * B * T - 1) // (NOFF * B * T)) * NOFF
CH = 256
traj = {}
for prec in ("fp32", "bf16"):
    m = dl.GpuRnn(V, H, 0, prec)
    m.set_params(*dl.init_uniform(V, H, int(g["init_seed"])))
    m.set_opt(None, None, None, 0.9995, 1e-6)
    m.trainer_init(ids, NOFF, B, T, 1.0)
    out = []
    for w0 in range(0, windows, CH):
        n = min(CH, windows - w0)
        if prec == "bf16" and w0 in (0, 1024, 3072):
            # the next window scored by this model and by an fp32 copy
            cur, hid = m.trainer_state()
            grp = (w0 % NOFF) * B
            pos = cur[None, grp:grp + B] + np.arange(T)[:, None]
            x, y = ids[pos % L], ids[(pos + 1) % L]
            wb = dl.WindowBatch(x, y, (y != 1).astype(np.uint8))
            h0 = hid[grp:grp + B]
            r16, _ = dl.bptt_run(m, wb, h0, 1.0 / (B * T), 1.0, compute_grads=False)
            f = dl.GpuRnn(V, H, 0, "fp32")
            f.set_params(*m.params())
            r32, _ = dl.bptt_run(f, wb, h0, 1.0 / (B * T), 1.0, compute_grads=False)
            f.close()
            print(f"window {w0}: bf16-model loss {r16.loss:.5f}, same params in fp32 "
                  f"{r32.loss:.5f}", flush=True)
        ls, _ = m.trainer_run(w0, n, eta)
        out.append(ls / n)
    traj[prec] = out
    print(prec, "mean", np.mean(out) if False else sum(o * min(CH, windows - i * CH)
                                                       for i, o in enumerate(out)) / windows,
          flush=True)
    m.close()
print("chunk  fp32   bf16")
for i, (a, b) in enumerate(zip(traj["fp32"], traj["bf16"])):
    print(f"{i * CH:5d} {a:.4f} {b:.4f} {100 * (b / a - 1):+.2f}%")
print("reference train loss", float(g["logs"][0][1]))
