mkdir -p gpurun_out; ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/nce_launches.csv python bench.py --loss nce --steps 2 --warmup 2 --no-e2e --secondary= --profile-steps 0 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import sys
sys.path.insert(0, "scripts")
from ncu_summary import launch_list
L = launch_list("gpurun_out/nce_launches.csv")
starts = [i for i, d in enumerate(L) if "k_window_build" in d["kernel"]]
win = L[starts[-1]:]
tot = 0
for d in win:
    t = d.get("gpu__time_duration.sum") or 0
    tot += t
    print(f"{t:8.1f} us  {d['kernel'][:100]}")
print("total", tot)
PY
