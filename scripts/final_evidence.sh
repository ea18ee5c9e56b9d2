#!/bin/bash
# Round-end evidence in one GPU call (1 GPU): the C3 launch list + ncu
# --set full captures (scripts/profile_c3.sh), their summary, the NCE launch
# list, the default bench line, the reference arm; results under
# gpurun_out/prof/ for profiles/.
#   scripts/final_evidence.sh <tag>
set -u
TAG=${1:-rXX}
mkdir -p gpurun_out/prof
bash scripts/profile_c3.sh $TAG > gpurun_out/prof/${TAG}_profile.log 2>&1
python scripts/ncu_summary.py $TAG > gpurun_out/prof/${TAG}_summary.log 2>&1
cp profiles/${TAG}_* gpurun_out/prof/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
bash scripts/nce_launches.sh > gpurun_out/prof/${TAG}_nce_launches.txt 2>&1
python - "$TAG" <<'PY'
import sys
sys.path.insert(0, "scripts")
from ncu_summary import launch_list
import csv
tag = sys.argv[1]
L = launch_list("gpurun_out/nce_launches.csv")
starts = [i for i, d in enumerate(L) if "k_window_build" in d["kernel"]]
win = L[starts[-1]:]
with open(f"gpurun_out/prof/{tag}_nce_launches_window.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["kernel", "duration_us", "dram_read_MB", "dram_write_MB"])
    for d in win:
        w.writerow([d["kernel"], d.get("gpu__time_duration.sum"), d.get("dram__bytes_read.sum"),
                    d.get("dram__bytes_write.sum")])
PY
python bench.py --steps 20 --warmup 5 2> gpurun_out/prof/${TAG}_bench.err | tail -1 > gpurun_out/prof/${TAG}_bench_c3.json
python bench.py --loss nce --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/prof/${TAG}_nce_bench_c3.json
python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 > gpurun_out/prof/${TAG}_reference_arm.json
ls -la gpurun_out/prof
