"""Tuning helper: alternate C3 bench runs under two environment settings and
report ms/window for each (run-to-run spread on a box is a few percent).
  python scripts/ab.py "DL_PAR_TAIL=0" "DL_PAR_TAIL=1" [rounds] [extra bench args]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
a, b = sys.argv[1], sys.argv[2]
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
extra = sys.argv[4:]
res = {a: [], b: []}
for r in range(rounds):
    for setting in (a, b):
        env = dict(os.environ)
        for kv in setting.split():
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "50",
                              "--warmup", "5", "--no-e2e", "--no-cpu-baseline", "--secondary="]
                             + extra, capture_output=True, text=True, env=env)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if not line:
            print(setting, "FAILED", out.stderr[-800:])
            continue
        d = json.loads(line[-1])
        res[setting].append(d["ms_per_step"])
        print(f"{setting:30s} {d['ms_per_step']:.4f} ms  clocks={d['clocks'].get('sm_mhz')} "
              f"{d['clocks'].get('reasons')}", flush=True)
for k, v in res.items():
    if v:
        print(f"{k:30s} mean {sum(v) / len(v):.4f} min {min(v):.4f}")
