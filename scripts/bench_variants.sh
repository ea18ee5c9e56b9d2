#!/bin/bash
# Tuning: run the C3 bench for the default build and each variants/<name>.
#   scripts/bench_variants.sh [bench args...]
ARGS=${*:-"--steps 50 --no-e2e --no-cpu-baseline --secondary="}
run() {
  local name=$1
  out=$(timeout 300 python bench.py $ARGS 2>&1 | grep '^{' | tail -1)
  python - "$name" "$out" <<'PY'
import json, sys
name, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    ph = d["roofline"]["phase_ms"]
    print(f"{name:12s} {d['value']:12.0f} words/s  {d['ms_per_step']:.4f} ms  " +
          " ".join(f"{k}={v:.3f}" for k, v in ph.items()))
except Exception as e:
    print(name, "FAILED", line[:300])
PY
}
run default
for d in variants/*/; do
  n=$(basename $d)
  DL_LIB_PATH=$PWD/variants/$n/libdesklm_cuda.so run $n
done
