#!/usr/bin/env python
"""RNNLM training throughput (words/sec, device-timed) on B200.

Default workload (BASELINE.json configs[2], the north-star target shape):
  C3 -- V = 64,000, H = 2,048, BPTT T = 16, B = 128 streams per GPU,
        noffset = 8, exact softmax, rmsprop, bf16 tensor cores (fp32
        masters); data-parallel over N GPUs with global minibatch 128*N.
A "step" is one truncated-BPTT window of the offset-stream schedule
(window build + forward + softmax + backward + rmsprop + hidden carry),
B*T words per GPU, exactly what Trainer::run_epoch does per window
(trainer.hpp:374-406).  Words include bos-target positions, as the
reference's tokens_per_sec does (trainer.hpp:250, :409).

  python bench.py [--gpus N --steps K --warmup W] [--config c1|c2|c3|c5]
  python bench.py --impl reference ...   # the reference CPU trainer
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = {"hbm_gbs": 6533.2, "bf16_tflops": 1679.5, "bf16_tflops_sustained": 1414.1}
try:
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        PEAKS.update(json.load(f))
except Exception:
    pass

CONFIGS = {
    # name: V, H, T, B(per GPU), noffset, L, data seed
    "c1": dict(V=10000, H=128, T=8, B=8, noffset=128, L=1_000_000, seed=1001,
               desc="RNNLM hidden=128, vocab=10K, BPTT=8, 1M-token stream"),
    "c2": dict(V=64000, H=1024, T=16, B=128, noffset=8, L=1 << 24, seed=2001,
               desc="RNNLM hidden=1024, vocab=64K full softmax, 128 streams"),
    "c3": dict(V=64000, H=2048, T=16, B=128, noffset=8, L=1 << 25, seed=3001,
               desc="RNNLM hidden=2048, vocab=64K, 128 streams/GPU, data-parallel"),
    # vocabulary-sharded output layer over the N GPUs (strong scaling: the
    # same B*T words per step, W_out rows split V/N per rank)
    "c4": dict(V=256000, H=4096, T=16, B=128, noffset=8, L=1 << 25, seed=4001, vshard=True,
               desc="RNNLM hidden=4096, vocab=256K, output softmax vocab-sharded over the GPUs"),
    # forward-only scoring (sharded_perplexity / n-best): a step = one
    # lock-step scoring step over S streams
    "c5": dict(V=64000, H=2048, T=1, B=1024, noffset=1, L=1 << 22, seed=5001, score=True,
               desc="perplexity scoring forward pass, hidden=2048, vocab=64K, 1024 streams"),
    # the bottleneck / tied-embedding model (compress.hpp) at the C3 shape
    # with a 512-wide projection: a step = one window through the C ABI
    # (dl_bn_train_window), host window arrays copied in every step
    "bn3": dict(V=64000, H=2048, P=512, T=16, B=128, noffset=8, L=1 << 22, seed=3001,
                bottleneck=True,
                desc="bottleneck RNNLM hidden=2048, projection=512, tied vocab=64K, 128 streams"),
}


def cpu_baseline_for(name: str, steps: int = 1):
    """The reference arm's measurement on a short bounded sample (a
    subprocess: `bench.py --impl reference --config name`), reported as
    this line's cpu_baseline."""
    try:
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference",
                            "--config", name, "--steps", str(steps), "--warmup", "0"],
                           capture_output=True, text=True, timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
        d = json.loads(line)
        if "unavailable" in d:
            return {"value": None, "error": d["unavailable"]}
        return dict(d["cpu_baseline"], same_config=d.get("same_config"))
    except Exception as ex:  # report, never fake
        return {"value": None, "error": str(ex)[:200]}


def measure_scoring(args, cfg, steps, warmup, cpu=True):
    """C5: sharded_perplexity scoring (eval.hpp:151-222 lock-step walk over S
    streams, exact softmax).  value: the scorer's kernels per step (CUDA
    events around each kernel class on the library stream, inputs resident);
    e2e: the public dl_score call with host arrays (H2D of the ids and
    targets, D2H of the per-token log-probs), CUDA events on the same stream."""
    import torch

    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200._lib import load
    V, H, S = cfg["V"], cfg["H"], cfg["B"]
    ids = synthetic_stream(cfg["seed"], V, cfg["L"])
    rng = np.random.default_rng(7)
    params = tuple(rng.uniform(-0.1, 0.1, s).astype(np.float32) for s in ((V, H), (H, H), (V, H)))
    model = dl.GpuRnn(V, H, 0, args.precision, 0)
    model.set_params(*params)
    n = len(ids) // S
    begin = np.arange(S) * n
    j = np.arange(steps + warmup)[:, None]
    x = ids[begin[None, :] + j].astype(np.uint32)
    y = ids[begin[None, :] + j + 1].astype(np.int64)
    t = np.where(y == 1, -1, y)
    stream = torch.cuda.ExternalStream(load().dl_cuda_stream(model.handle))
    for _ in range(max(1, min(warmup, 3))):  # warm-up: same shape (buffers, tensor maps)
        dl.score(model, x[warmup:], t[warmup:])
    launches0 = model.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        lp, tot, pred, _ = dl.score(model, x[warmup:], t[warmup:])
        e1.record(stream)
        torch.cuda.synchronize()
        time.sleep(0.25)
    launches = model.launch_count() - launches0
    e2e_ms = e0.elapsed_time(e1)
    # kernel-only time per step (profiling: events around each kernel class
    # over exactly one scoring bank of `bank` lock-step steps)
    bank = max(1, min(steps, 16384 // S))
    model.set_profiling(True)
    dl.score(model, x[warmup:warmup + bank], t[warmup:warmup + bank])
    phases = {k: model.kernel_ms(k) for k in ("recurrence_fwd", "logits", "softmax")}
    model.set_profiling(False)
    kern_ms = sum(v for v in phases.values() if v > 0) * steps / bank
    words = S * steps
    value = words / (kern_ms / 1000.0)
    fpw = 2 * H * V + 2 * H * H
    logit_ms = phases["logits"]
    logit_flops = 2.0 * bank * S * V * H
    achieved = logit_flops / (logit_ms / 1000.0) / 1e12
    out = {
        "metric": "scoring words/sec", "value": value, "unit": "words/s", "n_gpus": 1,
        "steps": steps, "warmup": warmup, "ms_per_step": kern_ms / steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.precision, "data": "synthetic",
        "config": {"workload": cfg["name"], "desc": cfg["desc"], "V": V, "H": H, "streams": S,
                   "l2": "inputs larger than L2 (W_out bf16 262 MB read per scoring bank)"},
        "flops_per_word": fpw, "mean_logprob": tot / max(pred, 1), "gpu_launches": launches,
        "clocks": clk.summary(),
        "roofline": {"bound": "tensor", "kernel": "tc_gemm[logits]", "unit": "TFLOP/s",
                     "achieved": achieved, "peak": PEAKS["bf16_tflops"],
                     "frac": achieved / PEAKS["bf16_tflops"], "traffic": None,
                     "peak_kind": "measured burst (MEASURED_PEAKS.json bf16_tflops)",
                     "algorithmic_flops_per_launch": logit_flops,
                     "step_frac_of_sustained_peak": value * fpw / 1e12
                     / PEAKS["bf16_tflops_sustained"], "phase_ms_per_bank": phases},
        "e2e": {"value": words / (e2e_ms / 1000.0), "unit": "words/s",
                "h2d_bytes_per_step": S * 12, "d2h_bytes_per_step": S * 8,
                "api": "dl_score (host ids / targets in, host per-token log-probs out), "
                       "CUDA events on the library stream"}}
    if cpu:
        out["cpu_baseline"] = cpu_baseline_for(cfg["name"])
    model.close()
    return out


def run_bottleneck(args, cfg):
    """Bottleneck model training words/s: bptt_run + bottleneck_update per
    window through dl_bn_train_window (device-timed with CUDA events on the
    library stream; each step copies its window in and its loss / h_final
    out, so value and e2e coincide)."""
    import torch

    import paper_1502_00512_b200 as dl
    from paper_1502_00512_b200 import bottleneck as bn
    from paper_1502_00512_b200._lib import load
    V, H, P, T, B = cfg["V"], cfg["H"], cfg["P"], cfg["T"], cfg["B"]
    ids = synthetic_stream(cfg["seed"], V, cfg["L"])
    rng = np.random.default_rng(7)
    params = tuple(rng.uniform(-0.1, 0.1, s).astype(np.float32)
                   for s in ((V, P), (P, H), (H, H), (H, P)))
    model = bn.GpuBottleneck(V, H, P, 0, args.precision, 0)
    model.set_params(*params)
    TB = T * B
    n = args.warmup + args.steps
    wins = []
    for i in range(n):
        s0 = (i * TB * 7) % (len(ids) - TB - 2)
        x = ids[s0:s0 + TB].reshape(T, B)
        y = ids[s0 + 1:s0 + 1 + TB].reshape(T, B)
        wins.append(dl.WindowBatch(x, y, (y != 1).astype(np.uint8)))
    h = np.full((B, H), 0.5, np.float32)
    stream = torch.cuda.ExternalStream(load().dl_bn_cuda_stream(model.handle))
    eta = 1e-3
    for wb in wins[: args.warmup]:
        _, h, _ = bn.bn_train_window(model, wb, h, 1.0 / TB, 1.0, eta)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = model.launch_count()
    loss = 0.0
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for wb in wins[args.warmup:]:
            r, h, _ = bn.bn_train_window(model, wb, h, 1.0 / TB, 1.0, eta)
            loss += r.loss
        e1.record(stream)
        torch.cuda.synchronize()
        time.sleep(0.25)
    ms = e0.elapsed_time(e1)
    launches = model.launch_count() - launches0
    value = TB * args.steps / (ms / 1000.0)
    # forward XU, Z (4PH), logits (2PV), recurrence (2H^2); backward dZ, gE
    # (4PV), dh_out, gD, gU, din (8PH), recurrence + gRec (4H^2)
    fpw = 6 * P * V + 6 * H * H + 12 * P * H
    peak = PEAKS["bf16_tflops_sustained"]
    cpu = None
    if not args.no_cpu_baseline:
        try:
            import oracle
            orc = oracle.Orc()
            Bs = 1
            t0 = time.perf_counter()
            wb = wins[0]
            r = orc.bn_bptt(params, 0, wb.inputs[:, :Bs], wb.targets[:, :Bs], wb.weights[:, :Bs],
                            np.full((Bs, H), 0.5, np.float32), 1.0 / (T * Bs), 1.0)
            st = (np.zeros(V, np.float32), np.zeros((P, H), np.float32),
                  np.zeros((H, H), np.float32), np.zeros((H, P), np.float32))
            orc.bn_update(params, st, r, 0.9995, 1e-6, eta)
            dt = time.perf_counter() - t0
            cpu = {"value": T * Bs / dt, "unit": "words/s", "cores": 1, "kind": "port",
                   "sample": f"one window T={T} x B={Bs} stream (bptt_run + bottleneck_update) "
                             f"at the full V/H/P, oracle C restatement, {dt:.1f} s"}
        except Exception as ex:
            cpu = {"value": None, "error": str(ex)[:200]}
    print(json.dumps({
        "metric": "training words/sec", "value": value, "unit": "words/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": args.precision, "data": "synthetic",
        "config": {"workload": "bn3", "desc": cfg["desc"], "V": V, "H": H, "P": P, "T": T,
                   "B_per_gpu": B, "loss": "exact softmax", "model": "bottleneck (tied E)"},
        "flops_per_word": fpw, "mean_window_loss": loss / args.steps, "gpu_launches": launches,
        "clocks": clk.summary(),
        "roofline": {"bound": "tensor", "kernel": "whole window (GEMMs + recurrence + update)",
                     "unit": "TFLOP/s", "achieved": value * fpw / 1e12, "peak": peak,
                     "frac": value * fpw / 1e12 / peak, "traffic": None,
                     "peak_kind": "measured sustained (MEASURED_PEAKS.json)"},
        "e2e": {"value": value, "unit": "words/s", "h2d_bytes_per_step": TB * 9 + B * H * 4,
                "d2h_bytes_per_step": B * H * 4 + 16,
                "api": "dl_bn_train_window per step, host window arrays"},
        "cpu_baseline": cpu}), flush=True)


def synthetic_stream(seed: int, V: int, L: int) -> np.ndarray:
    """Sentences <s> w.. </s> of 1..12 words, ids 3 + min(u1, u2) over [3, V)
    -- the shape of the reference's random_stream fixture
    (tests/oracles/helpers.hpp:36-52), generated vectorised."""
    rng = np.random.default_rng(seed)
    out = np.empty(L + 64, np.uint32)
    n = 0
    while n < L:
        k = 65536
        lens = rng.integers(1, 13, k)
        tot = int(lens.sum()) + 2 * k
        body = np.minimum(rng.integers(0, V - 3, tot), rng.integers(0, V - 3, tot)) + 3
        ends = np.cumsum(lens + 2)
        starts = ends - lens - 2
        body[starts] = 1
        body[ends - 1] = 2
        take = min(tot, L + 64 - n)
        out[n:n + take] = body[:take]
        n += take
    return out[:L]


def flops_per_word(V, H, nce_k=0):
    """6*H*V + 6*H^2: forward logits + recurrence, dS.W_out + dW_out, the
    recurrent backward and dW_rec.  NCE: the output layer
    touches k + 1 rows per word instead of V."""
    return 6 * H * (nce_k + 1 if nce_k else V) + 6 * H * H


class ClockSampler:
    def __init__(self, index: int):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML initialisation) must not overlap the
            # short timed region: wait for its first sample (<= 3 s)
            t0 = time.time()
            while not self.samples and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 5 + i and s[5 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# Bounded sample of each workload for the reference CPU timer: B streams x
# Ts unrolled steps per window (softmax training), or S slices (scoring).
# The reference's dW_out product (matmul_tn_add, mat.hpp:168-184) is single-
# threaded and streams the whole V x H gradient once per position, so at
# the C2-C4 shapes one window position costs seconds: T is cut to 1 (B
# stays the config's, except C4's 256K x 4K gradient).
REF_SAMPLE = {"c1": dict(T=8, B=8), "c2": dict(T=1, B=128), "c3": dict(T=1, B=128),
              "c4": dict(T=1, B=16), "c5": dict(S=1024), "bn3": dict(T=1, B=1)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    name = line.split(":", 1)[1].strip()
                    break
            else:
                name = "unknown"
        with open("/proc/cpuinfo") as f:
            txt = f.read()
        fam = [l.split(":")[1].strip() for l in txt.splitlines() if l.startswith("model\t")]
        return f"{name} (model {fam[0] if fam else '?'}), {os.cpu_count()} logical CPUs"
    except Exception:
        return "unknown"


def run_reference(args, cfg):
    """The reference's own CPU implementation of the path, timed in-process:
    oracle/_ref/ref_bench (the unmodified /root/reference headers built with
    the reference's flags -O3 -march=<host ISA>, threads = all host CPUs)
    runs Trainer::run_epoch's window body -- bptt_run + rmsprop_update on
    resident parameters -- or sharded_perplexity, for exactly --warmup +
    --steps steps of a bounded sample of the workload (REF_SAMPLE)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    V, H, T = cfg["V"], cfg["H"], cfg["T"]
    smp = REF_SAMPLE[cfg["name"]]
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    score = bool(cfg.get("score"))
    if cfg.get("bottleneck"):
        return run_reference_bn(args, cfg, cores)
    if not os.path.exists(exe):
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/ref_bench not built (needs /root/reference at build time)"}))
        return
    if score:
        S = smp["S"]
        argv = [exe, "score", str(V), str(H), str(S), "-", str(args.steps), str(args.warmup),
                str(cores)]
        words_per_step = S
        sample = (f"sharded_perplexity over S={S} slices (the C5 config), {args.steps} timed "
                  f"lock-step scoring steps after {args.warmup} warm-up steps, threads={cores}")
        metric = "scoring words/sec"
    else:
        Ts, Bs = smp["T"], smp["B"]
        argv = [exe, "train", str(V), str(H), str(Ts), str(Bs), str(args.steps), str(args.warmup),
                str(cores)]
        words_per_step = Ts * Bs
        sample = (f"window-sampled: {args.steps} timed windows (+{args.warmup} warm-up) of "
                  f"B={Bs} streams x T={Ts} at V={V}, H={H} (config: B={cfg['B']}, T={T}); "
                  f"bptt_run(StandardAdapter, softmax) + rmsprop_update in-process on resident "
                  f"params, threads={cores}")
        metric = "training words/sec"
    r = subprocess.run(argv, capture_output=True, text=True)
    if r.returncode != 0:
        print(json.dumps({"impl": "reference", "unavailable": f"ref_bench failed: "
                          f"{r.stderr.strip()[:200]}"}))
        return
    res = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    times = res["step_s"]
    value = words_per_step * len(times) / sum(times)
    same = score or (smp.get("T") == T and smp.get("B") == cfg["B"])
    print(json.dumps({
        "metric": metric, "value": value, "unit": "words/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": 1000 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 accumulate)",
        "data": "synthetic",
        "config": {"workload": cfg["name"], "desc": cfg["desc"], "V": V, "H": H, "T": T,
                   "B_per_gpu": cfg["B"]},
        "same_config": same,
        "cpu_baseline": {"value": value, "unit": "words/s", "cores": cores, "kind": "reference",
                         "sample": sample, "cpu": cpu_model(),
                         "build": "g++ -O3 -march=sapphirerapids (the GPU host's native ISA)"},
        "e2e": {"value": value, "unit": "words/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def run_reference_bn(args, cfg, cores):
    """Bottleneck model reference arm: bptt_run(BottleneckAdapter) +
    bottleneck_update through the compiled reference shim (or the oracle)."""
    import oracle
    try:
        ref, kind = oracle.Ref(), "reference"
    except FileNotFoundError:
        ref, kind = oracle.Orc(), "port"
    V, H, P, T = cfg["V"], cfg["H"], cfg["P"], cfg["T"]
    Bs, Ts = 1, 1
    ids = synthetic_stream(cfg["seed"], V, 1 << 16)
    rng = np.random.default_rng(1)
    params = tuple(rng.uniform(-0.1, 0.1, s).astype(np.float32)
                   for s in ((V, P), (P, H), (H, H), (H, P)))
    state = (np.zeros(V, np.float32), np.zeros((P, H), np.float32),
             np.zeros((H, H), np.float32), np.zeros((H, P), np.float32))
    h0 = np.full((Bs, H), 0.5, np.float32)
    times = []
    for i in range(args.warmup + args.steps):
        s0 = i * Bs * Ts
        x = ids[s0:s0 + Ts * Bs].reshape(Ts, Bs)
        y = ids[s0 + 1:s0 + 1 + Ts * Bs].reshape(Ts, Bs)
        w = (y != 1).astype(np.uint8)
        t0 = time.perf_counter()
        g = ref.bn_bptt(params, 0, x, y, w, h0, 1.0 / (Bs * Ts), 1.0)
        params, state, _ = ref.bn_update(params, state, g, 0.9995, 1e-6, 0.05)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    value = Bs * Ts * len(times) / sum(times)
    print(json.dumps({
        "metric": "training words/sec", "value": value, "unit": "words/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": 1000 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 accumulate)",
        "data": "synthetic", "config": {"workload": cfg["name"], "V": V, "H": H, "P": P},
        "cpu_baseline": {"value": value, "unit": "words/s", "cores": 1, "kind": kind,
                         "sample": f"{len(times)} windows of B={Bs} x T={Ts} (bptt_run("
                                   f"BottleneckAdapter) + bottleneck_update), threads=1",
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "words/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def measure_training(args, cfg, world, rank, local, steps, warmup, dist=None, cpu=True):
    """Training words/s of one configuration: a step is one window of the
    offset-stream schedule run by the device trainer (dl_trainer_run),
    CUDA events on the library stream, max over ranks; then per-kernel times,
    the roofline of the dominant kernel, and the e2e figure through
    dl_train_window with page-locked host arrays."""
    import torch

    import paper_1502_00512_b200 as dl
    V, H, T, B, noffset = cfg["V"], cfg["H"], cfg["T"], cfg["B"], cfg["noffset"]
    L = cfg["L"]
    ids = synthetic_stream(cfg["seed"], V, L)
    rng = np.random.default_rng(7)  # random-init weights, init_uniform range 0.1
    params = tuple(rng.uniform(-0.1, 0.1, s).astype(np.float32)
                   for s in ((V, H), (H, H), (V, H)))
    model = dl.GpuRnn(V, H, 0, args.precision, local)
    if world > 1:
        uid = [dl.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        model.comm_init(uid[0], world, rank)
        if cfg.get("vshard"):
            model.set_vocab_shard(True)
        elif args.dp_mode == "vocab":
            # data-parallel streams, vocabulary-parallel output layer: no
            # V x H gradient on the links, the W_out update split N ways
            model.set_vocab_shard("dp")
    model.set_params(*params)
    del params
    model.set_opt(None, None, None, 0.9995, 1e-6)
    if args.loss == "nce":
        counts = np.bincount(ids[ids != 1], minlength=V).astype(np.float64)
        model.set_loss_mode(0)
        model.set_noise(counts, args.nce_k, 1e-8)
        model.set_rng_state(dl.rng_seed_state(1))
    model.trainer_init(ids, noffset, B, T, 1.0)
    eta = 1e-3
    stream = torch.cuda.ExternalStream(dl._lib.load().dl_cuda_stream(model.handle))

    def barrier():
        if world > 1:
            dist.barrier()

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # clocks are sampled from before the warm-up through the timed region
    # (nvidia-smi's 100 ms period would otherwise miss a short timed region)
    with ClockSampler(local) as clk:
        # warm-up (also captures the per-window CUDA graphs)
        model.trainer_run(0, warmup, eta)
        torch.cuda.synchronize()
        launches0 = model.launch_count()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        loss_sum, skipped = model.trainer_run(warmup, steps, eta)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        time.sleep(0.25)
    ms = e0.elapsed_time(e1)
    launches = model.launch_count() - launches0
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    vshard = bool(cfg.get("vshard"))
    # data parallel: every rank trains its own B streams; vocabulary-sharded:
    # all ranks cooperate on the same B streams
    words = (1 if vshard else world) * B * T * steps
    value = words / (ms / 1000.0)
    fpw = flops_per_word(V, H, args.nce_k if args.loss == "nce" else 0)

    # per-kernel device times (eager launches + CUDA events on the library
    # stream) -> roofline of the dominant kernel
    model.set_profiling(True)
    model.trainer_run(warmup + steps, args.profile_steps, eta)
    phases = {}
    for name in ("recurrence_fwd", "logits", "softmax", "dh", "dw_out", "nce_loss", "nce_dh",
                 "recurrence_bwd", "dw_rec", "embed_grad", "nce_out_rows", "rmsprop",
                 "rmsprop_out", "vocab_exchange"):
        v = model.kernel_ms(name)
        if v >= 0:
            phases[name] = v
    model.set_profiling(False)
    TB = T * B
    # W_out rows on this GPU; with the vocabulary-parallel DP output layer
    # each GPU scores world x TB rows against V / world
    dpv = world > 1 and args.dp_mode == "vocab" and not vshard
    Vloc = V // world if (vshard or dpv) else V
    TBo = TB * world if dpv else TB
    gemm_flops = {"logits": 2.0 * TBo * Vloc * H, "dh": 2.0 * TBo * Vloc * H,
                  "dw_out": 2.0 * TBo * Vloc * H}
    dom = max(gemm_flops, key=lambda k: phases.get(k, 0.0))
    dom_ms = phases.get(dom, float("nan"))
    achieved = gemm_flops[dom] / (dom_ms / 1000.0) / 1e12
    # the per-kernel times are CUDA events around single launches inside
    # the step: the burst peak applies; the whole step is held against the
    # sustained peak
    peak = PEAKS["bf16_tflops"]
    step_ms = ms / steps
    traffic, traffic_src = None, None  # DRAM bytes per launch from the committed ncu capture
    try:
        import glob
        for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_summary.json"))):
            with open(path) as f:
                sm = json.load(f).get("dominant_kernel_for_bench_roofline", {})
            if sm.get("kernel") == f"tc_gemm[{dom}]" and sm.get("config") == cfg["name"]:
                traffic, traffic_src = sm["traffic_bytes_per_launch"], os.path.basename(path)
    except Exception:
        pass
    roofline = {"bound": "tensor", "kernel": f"tc_gemm[{dom}]", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "traffic_source": traffic_src,
                "peak_kind": "measured burst (MEASURED_PEAKS.json bf16_tflops)",
                "algorithmic_flops_per_launch": gemm_flops[dom],
                "step_frac_of_sustained_peak": value / world * fpw / 1e12
                / PEAKS["bf16_tflops_sustained"],
                "step_frac_of_burst_peak": value / world * fpw / 1e12 / PEAKS["bf16_tflops"],
                "phase_ms": phases}
    if dom == "dw_out":
        roofline["note"] = ("dW_out GEMM with the dense W_out rmsprop fused into its epilogue "
                            "(+10 B/elem of W_out: fp32 master read+write, bf16 shadow write)")

    # end-to-end through the public API with host buffers: dl_train_window
    # per step (H2D of the window ids/targets/mask/h0 from page-locked host
    # memory, bptt_run + rmsprop_update, D2H of loss, positions, applied and
    # h_final), CUDA events on the library stream around all the calls
    e2e = None
    # (NCE: single-rank windows only through this call; the noise of each
    # window is drawn by the library from the context's generator)
    if args.e2e and (args.loss == "softmax" or world == 1):
        def pinned(shape, dtype):
            return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()

        n_e2e = steps + 3
        wins = []
        for i in range(n_e2e):
            s0 = (i * TB * 7) % (L - TB - 2)
            x, y, w = pinned((T, B), torch.int32), pinned((T, B), torch.int32), \
                pinned((T, B), torch.uint8)
            x[:] = ids[s0:s0 + TB].reshape(T, B)
            y[:] = ids[s0 + 1:s0 + 1 + TB].reshape(T, B)
            w[:] = y != 1
            wins.append(dl.WindowBatch(x.view(np.uint32), y.view(np.uint32), w))
        hbuf = [pinned((B, H), torch.float32) for _ in range(2)]
        hbuf[0][:] = 0.5
        for i in range(3):  # warm-up
            dl.train_window(model, wins[i], hbuf[i % 2], 1.0 / TB, 1.0, eta,
                            h_final=hbuf[(i + 1) % 2])
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        for i, wb in enumerate(wins[3:]):
            dl.train_window(model, wb, hbuf[(i + 1) % 2], 1.0 / TB, 1.0, eta,
                            h_final=hbuf[i % 2])
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        dt = e0.elapsed_time(e1) / 1000.0
        if world > 1:
            tt = torch.tensor([dt, wall], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt, wall = float(tt[0].item()), float(tt[1].item())
        e2e = {"value": world * TB * steps / dt, "unit": "words/s", "steps": steps,
               "h2d_bytes_per_step": TB * 9 + B * H * 4,
               "d2h_bytes_per_step": B * H * 4 + 8 + 8 + 4,
               "wall_clock_value": world * TB * steps / wall,
               "api": "dl_train_window (bptt_run + rmsprop_update), page-locked host arrays, "
                      "CUDA events on the library stream"}

    cpu_b = None
    if cpu and rank == 0 and world == 1:
        cpu_b = cpu_baseline_for(cfg["name"])
    out = {"metric": "training words/sec", "value": value, "unit": "words/s",
           "n_gpus": world, "steps": steps, "warmup": warmup,
           "ms_per_step": step_ms, "higher_is_better": True,
           "scaling": "strong" if vshard else "weak",
           "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
           "config": {"workload": cfg["name"], "desc": cfg["desc"], "V": V, "H": H,
                      "T": T, "B_per_gpu": B,
                      "global_minibatch": B if vshard else B * world,
                      "noffset": noffset, "L": L,
                      "loss": ("exact softmax" if args.loss == "softmax"
                               else f"NCE k={args.nce_k}"),
                      "optimizer": "rmsprop (per-word W_in/W_out scalars)",
                      "parallelism": (f"vocab{world}" if vshard else
                                      f"dp{world}+vocab-parallel-output"
                                      if world > 1 and args.dp_mode == "vocab"
                                      else f"dp{world}"),
                      "l2": "inputs larger than L2 (W_out bf16 + fp32 master, "
                            f"{6 * Vloc * H / 1e6:.0f} MB, streamed every window)"},
           "flops_per_word": fpw, "mean_window_loss": loss_sum / steps,
           "skipped_updates": skipped, "gpu_launches": launches,
           "clocks": clk.summary(), "roofline": roofline, "e2e": e2e,
           "cpu_baseline": cpu_b}
    model.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32", "tf32x3"])
    ap.add_argument("--loss", default="softmax", choices=["softmax", "nce"],
                    help="output layer: exact softmax (the north-star path) or NCE "
                         "(LossMode::kNce, the reference's default training mode)")
    ap.add_argument("--nce-k", type=int, default=64)
    ap.add_argument("--dp-mode", default="vocab", choices=["vocab", "dense"],
                    help="N>1 data parallel: vocabulary-parallel output layer (default) or "
                         "the dense dW_out allreduce")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--profile-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--secondary", default="c2,c5,c4",
                    help="configs measured after the headline one (N=1 only) and reported "
                         "in the line's `secondary` list; '' for none")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config], name=args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    if cfg.get("bottleneck"):
        run_bottleneck(args, cfg)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cpu = not args.no_cpu_baseline
    if cfg.get("score"):
        out = measure_scoring(args, cfg, args.steps, args.warmup, cpu=cpu)
    else:
        out = measure_training(args, cfg, world, rank, local, args.steps, args.warmup, dist,
                               cpu=cpu)
    if world == 1 and args.secondary:
        sec = []
        for name in [n for n in args.secondary.split(",") if n and n != args.config]:
            c2 = dict(CONFIGS[name], name=name)
            try:
                if c2.get("score"):
                    sec.append(measure_scoring(args, c2, args.steps, args.warmup, cpu=cpu))
                else:
                    sec.append(measure_training(args, c2, 1, 0, local, args.steps, args.warmup,
                                                cpu=cpu))
            except Exception as ex:  # report, never fake
                sec.append({"config": {"workload": name}, "error": str(ex)[:300]})
            torch.cuda.empty_cache()
        out["secondary"] = sec
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
