#!/bin/bash
# ncu launch list (duration + DRAM bytes) of 2 C3 windows after warm-up;
# prints the last window's kernels.  scripts/launches.sh <tag>
TAG=${1:-tmp}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --secondary= --profile-steps 0 --no-cpu-baseline \
    > gpurun_out/${TAG}_launches.log 2>&1
python - "$TAG" <<'PY'
import sys
sys.path.insert(0, "scripts")
from ncu_summary import launch_list
L = launch_list(f"gpurun_out/{sys.argv[1]}_launches.csv")
starts = [i for i, d in enumerate(L) if "k_window_build" in d["kernel"]]
win = L[starts[-1]:]
tot = 0
for d in win:
    t = d.get("gpu__time_duration.sum") or 0
    tot += t
    print(f"{t:8.1f} us  R {d.get('dram__bytes_read.sum',0):7.1f} W {d.get('dram__bytes_write.sum',0):7.1f} MB  {d['kernel'][:90]}")
print(f"total {tot:.1f} us")
PY
