"""Diagnostics: accuracy of the fp32-mode GEMMs vs float64 (argv[1]: tf32x3 | fp32)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_1502_00512_b200 as dl
from paper_1502_00512_b200._lib import load
m = dl.GpuRnn(16, 8, 0, sys.argv[1] if len(sys.argv) > 1 else "tf32x3")
rng = np.random.default_rng(0)
for (M, N, K, dist) in [(128, 128, 10000, "sym"), (128, 128, 10000, "pos"), (64, 128, 10000, "sym"),
                        (128, 128, 64000, "pos"), (256, 256, 2048, "sym")]:
    if dist == "sym":
        A = rng.uniform(-1, 1, (M, K)).astype(np.float32); B = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    else:
        A = rng.uniform(0, 1, (M, K)).astype(np.float32); B = rng.uniform(0, 1, (N, K)).astype(np.float32)
    out = np.empty((M, N), np.float32)
    rc = load().dl_test_gemm(m.handle, M, N, K, 0, 0, A.ctypes.data, B.ctypes.data, out.ctypes.data, 1, None)
    assert rc == 0, rc
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    err = (out - ref)
    scale = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64).T
    print(f"M{M} N{N} K{K} {dist}: max|err|/sum|ab| {np.max(np.abs(err)/scale):.3e} "
          f"mean(err/sum|ab|) {np.mean(err/scale):.3e} max rel {np.max(np.abs(err)/np.abs(ref)):.3e}")
