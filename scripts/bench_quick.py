#!/usr/bin/env python
"""Tuning helper: run bench.py (C3, short) and print words/s + per-phase ms."""
import json
import subprocess
import sys

args = sys.argv[1:] or ["--steps", "50", "--e2e-steps", "0", "--no-cpu-baseline"]
out = subprocess.run([sys.executable, "bench.py"] + args, capture_output=True, text=True)
line = [l for l in out.stdout.splitlines() if l.startswith("{")]
if not line:
    print("FAILED", out.stdout[-2000:], out.stderr[-3000:])
    sys.exit(1)
d = json.loads(line[-1])
ph = d.get("roofline", {}).get("phase_ms", {})
print(f"{d['value']:.0f} words/s {d['ms_per_step']:.4f} ms/step clocks={d.get('clocks')}")
print(" ".join(f"{k}={v:.3f}" for k, v in ph.items()))
