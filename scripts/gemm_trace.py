"""Epilogue phase timings of the fused dW_out + rmsprop GEMM at C3 (DL_GEMM_TRACE)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DL_GEMM_TRACE"] = "1"
import numpy as np
import paper_1502_00512_b200 as dl
V, H, T, B = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (64000, 2048, 16, 128)))
rng = np.random.default_rng(0)
m = dl.GpuRnn(V, H, 0, "bf16")
m.set_params(*(rng.uniform(-0.1, 0.1, s).astype(np.float32) for s in ((V, H), (H, H), (V, H))))
x = rng.integers(3, V, (T, B)).astype(np.uint32)
y = rng.integers(3, V, (T, B)).astype(np.uint32)
wb = dl.WindowBatch(x, y, np.ones((T, B), np.uint8))
h0 = np.full((B, H), 0.5, np.float32)
for _ in range(3):
    dl.train_window(m, wb, h0, 1.0 / (T * B), 1.0, 1e-3)
