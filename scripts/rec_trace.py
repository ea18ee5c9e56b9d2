"""Per-step phase timings of the persistent recurrence at C3 (DL_REC_TRACE)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["DL_REC_TRACE"] = "1"
import numpy as np
import paper_1502_00512_b200 as dl
V, H, T, B = 64000, 2048, 16, 128
rng = np.random.default_rng(0)
m = dl.GpuRnn(V, H, 0, "bf16")
m.set_params(*(rng.uniform(-0.1, 0.1, s).astype(np.float32) for s in ((V, H), (H, H), (V, H))))
x = rng.integers(3, V, (T, B)).astype(np.uint32)
y = rng.integers(3, V, (T, B)).astype(np.uint32)
wb = dl.WindowBatch(x, y, np.ones((T, B), np.uint8))
h0 = np.full((B, H), 0.5, np.float32)
for _ in range(3):
    dl.bptt_run(m, wb, h0, 1.0 / (T * B), 1.0)
