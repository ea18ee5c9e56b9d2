"""Diagnostics: per-call cost of dl_train_window around the device window --
the C3 window vs a tiny model (V = 1,000, H = 128, same T x B) whose device
time is negligible, with page-locked host buffers as bench.py's e2e leg."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1502_00512_b200 as dl


def run(V, H, T=16, B=128, n=30):
    def pinned(shape, dtype):
        return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()
    m = dl.GpuRnn(V, H, 0, "bf16")
    rng = np.random.default_rng(0)
    m.set_params(*(rng.uniform(-0.1, 0.1, s).astype(np.float32) for s in ((V, H), (H, H), (V, H))))
    m.set_opt(None, None, None, 0.9995, 1e-6)
    x = pinned((T, B), torch.int32); x[:] = rng.integers(2, V, (T, B))
    y = pinned((T, B), torch.int32); y[:] = rng.integers(2, V, (T, B))
    w = pinned((T, B), torch.uint8); w[:] = 1
    wb = dl.WindowBatch(x.view(np.uint32), y.view(np.uint32), w)
    h = [pinned((B, H), torch.float32) for _ in range(2)]
    h[0][:] = 0.5
    for i in range(5):
        dl.train_window(m, wb, h[i % 2], 1.0 / (T * B), 1.0, 1e-3, h_final=h[(i + 1) % 2])
    t0 = time.perf_counter()
    for i in range(n):
        dl.train_window(m, wb, h[i % 2], 1.0 / (T * B), 1.0, 1e-3, h_final=h[(i + 1) % 2])
    dt = (time.perf_counter() - t0) / n
    m.close()
    return dt


print(f"tiny V=1000 H=128: {1e6 * run(1000, 128):.1f} us per call")
print(f"tiny V=1000 H=2048: {1e6 * run(1000, 2048):.1f} us per call")
print(f"C3 V=64000 H=2048: {1e6 * run(64000, 2048):.1f} us per call")
