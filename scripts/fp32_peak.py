"""Microbenchmark of the fp32 SIMT (no TF32) GEMM peak on this B200 -- the
roofline of the fp32 parity mode ("fp32-SIMT peak must be
microbenchmarked and recorded").  cuBLAS SGEMM via torch with TF32 off, and
this repository's own SIMT kernel (dl_test_gemm) at the same shape."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

torch.backends.cuda.matmul.allow_tf32 = False
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 10
for _ in range(reps):
    a @ b
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
cublas = 2 * n ** 3 / (ms / 1e3) / 1e12

import paper_1502_00512_b200 as dl  # noqa: E402
from paper_1502_00512_b200._lib import load  # noqa: E402
import ctypes as C  # noqa: E402
m = dl.GpuRnn(16, 8, 0, "fp32")
M = N = K = 4096
A = np.random.default_rng(0).standard_normal((M, K)).astype(np.float32)
B = np.random.default_rng(1).standard_normal((N, K)).astype(np.float32)
out = np.empty((M, N), np.float32)
lib = load()
lib.dl_test_gemm(m.handle, M, N, K, 0, 0, A.ctypes.data, B.ctypes.data, out.ctypes.data, 1, None)
t0 = time.perf_counter()
lib.dl_test_gemm(m.handle, M, N, K, 0, 0, A.ctypes.data, B.ctypes.data, out.ctypes.data, 1, None)
dt = time.perf_counter() - t0
print(json.dumps({"cublas_sgemm_fp32_tflops": cublas, "n": n,
                  "own_simt_gemm_tflops_incl_host_copies": 2 * M * N * K / dt / 1e12,
                  "note": "TF32 disabled; the repository's SIMT number includes the H2D/D2H "
                          "copies of dl_test_gemm (a lower bound)"}))
