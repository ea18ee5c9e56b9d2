"""Diagnostics: per-tile phase trace of the fused dW_out + rmsprop epilogue
(DL_GEMM_TRACE) at the C3 shape through dl_train_window."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DL_GEMM_TRACE"] = "1"
import numpy as np
import paper_1502_00512_b200 as dl
V, H, T, B = 64000, 2048, 16, 128
rng = np.random.default_rng(0)
params = tuple(rng.uniform(-0.1, 0.1, s).astype(np.float32) for s in ((V, H), (H, H), (V, H)))
m = dl.GpuRnn(V, H, 0, "bf16")
m.set_params(*params)
m.set_opt(None, None, None, 0.9995, 1e-6)
x = rng.integers(3, V, (T, B)).astype(np.uint32)
y = rng.integers(3, V, (T, B)).astype(np.uint32)
w = np.ones((T, B), np.uint8)
h = np.full((B, H), 0.5, np.float32)
for i in range(4):
    r, h, ok = dl.train_window(m, dl.WindowBatch(x, y, w), h, 1.0 / (T * B), 1.0, 1e-3)
print("done", r.loss)
