#!/usr/bin/env python
"""Summarise the ncu captures of scripts/profile_c3.sh into profiles/.

  python scripts/ncu_summary.py <tag>

Reads gpurun_out/<tag>_launches.csv (every launch: duration + DRAM bytes)
and gpurun_out/<tag>_prof_*.ncu-rep (--set full), writes
profiles/<tag>_launches_window.csv (the last window's launch list) and
profiles/<tag>_ncu_summary.json (per-kernel duration, DRAM traffic, tensor
pipe / DRAM utilisation, SM clock under the profiler).
"""
import collections
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1.0),
    "dram_read_MB": ("dram__bytes_read.sum", 1.0),
    "dram_write_MB": ("dram__bytes_write.sum", 1.0),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "sm_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
}


def to_float(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return None


def launch_list(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                              "Metric Unit"))
    out = collections.OrderedDict()
    for r in rows[i + 1:]:
        if len(r) < len(hdr):
            continue
        d = out.setdefault(r[0], {"kernel": r[ki]})
        v = to_float(r[vi])
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3,
                 "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(r[ui], 1.0)
        d[r[mi]] = v * scale if v is not None else None
    return list(out.values())


def full_captures(tag):
    res = []
    for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", f"{tag}_prof_*.ncu-rep"))):
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            k = {"kernel": d["Kernel Name"]}
            for name, (m, _) in METRICS.items():
                if m not in d:
                    continue
                v = to_float(d[m])
                unit = u.get(m, "")
                if v is not None and name.endswith("_MB"):
                    v *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
                if v is not None and name == "duration_us":
                    v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1.0)
                if v is not None and name == "sm_ghz":
                    v *= {"cycle/nsecond": 1.0, "cycle/usecond": 1e-3, "cycle/second": 1e-9}.get(
                        unit, 1.0)
                k[name] = v
            res.append(k)
    return res


def main():
    tag = sys.argv[1]
    L = launch_list(os.path.join(ROOT, "gpurun_out", f"{tag}_launches.csv"))
    # the last window: from the last k_window_build launch to the end
    starts = [i for i, d in enumerate(L) if "k_window_build" in d["kernel"]]
    win = L[starts[-1]:] if starts else L
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches_window.csv"), "w") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "duration_us", "dram_read_MB", "dram_write_MB"])
        for d in win:
            w.writerow([d["kernel"][:120], round(d.get("gpu__time_duration.sum") or 0, 2),
                        round(d.get("dram__bytes_read.sum") or 0, 2),
                        round(d.get("dram__bytes_write.sum") or 0, 2)])
    total = sum(d.get("gpu__time_duration.sum") or 0 for d in win)
    kernels = full_captures(tag)
    # the GEMM each pair-kernel instantiation serves in the C3 window
    # (<A-major, B-major, fused rmsprop[, XF]>)
    roles = {"tc_gemm2_kernel<0, 0, 0": "tc_gemm[logits]", "tc_gemm2_kernel<0, 1, 0": "tc_gemm[dh]",
             "tc_gemm2_kernel<1, 1, 1": "tc_gemm[dw_out]", "tc_gemm2_kernel<1, 1, 0": "tc_gemm[dw_rec]"}
    for k in kernels:
        for pat, role in roles.items():
            i = k["kernel"].find(pat)
            if i >= 0 and k["kernel"][i + len(pat)] in ",>":
                k["role"] = role
    gemms = [k for k in kernels if k.get("role") in ("tc_gemm[logits]", "tc_gemm[dh]",
                                                     "tc_gemm[dw_out]")]
    dom = None
    if gemms:
        d = max(gemms, key=lambda k: k.get("duration_us") or 0)
        dom = {"kernel": d["role"], "config": "c3",
               "traffic_bytes_per_launch": int(((d.get("dram_read_MB") or 0) +
                                                (d.get("dram_write_MB") or 0)) * 1e6),
               "duration_us_under_ncu": d.get("duration_us")}
    summary = {"tag": tag, "window_launches": len(win), "window_us_serialised_cold": total,
               "dominant_kernel_for_bench_roofline": dom,
               "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_* (launch list) and "
                         "--set full --clock-control none (captures) of scripts/profile_c3.sh",
               "kernels": kernels}
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
