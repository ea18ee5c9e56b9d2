"""Tuning helper: per-phase device time of the C5 scoring step (1,024 streams,
H=2,048, V=64,000; banks of 4 steps per logits GEMM)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1502_00512_b200 as dl
V, H, S, steps = 64000, 2048, 1024, 16
rng = np.random.default_rng(0)
m = dl.GpuRnn(V, H, 0, "bf16")
m.set_params(*(rng.uniform(-0.1, 0.1, s).astype(np.float32) for s in ((V, H), (H, H), (V, H))))
x = rng.integers(3, V, (steps, S)).astype(np.uint32)
t = rng.integers(3, V, (steps, S)).astype(np.int64)
dl.score(m, x, t)
m.set_profiling(True)
dl.score(m, x, t)
for k in ("recurrence_fwd", "logits", "softmax"):
    print(k, round(m.kernel_ms(k), 4), "ms per call")
