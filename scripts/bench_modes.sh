#!/bin/bash
# Tuning: C3 bench under each W_out-update placement (env knobs of runtime.cu).
ARGS=${*:-"--steps 50 --e2e-steps 0 --no-cpu-baseline"}
for mode in "DL_FUSE_OUT=1" "DL_FUSE_OUT=0" "DL_FUSE_OUT=0 DL_FORK_LATE=1" "DL_FUSE_OUT=0 DL_FORK_OUT=1"; do
  out=$(env $mode timeout 300 python bench.py $ARGS 2>&1 | grep '^{' | tail -1)
  python -c "
import json,sys
d=json.loads(sys.argv[2]); ph=d['roofline']['phase_ms']
print(f\"{sys.argv[1]:34s} {d['value']:10.0f} w/s {d['ms_per_step']:.4f} ms \" + ' '.join(f'{k}={v:.3f}' for k,v in ph.items()))
" "$mode" "$out" || echo "$mode FAILED $out"
done
