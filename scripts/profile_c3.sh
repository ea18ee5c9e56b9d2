#!/bin/bash
# ncu evidence for the C3 training window (run under gpurun, 1 GPU).
#   scripts/profile_c3.sh <tag>
# 1. launch list of every kernel of 2 windows after warm-up (cold-cache,
#    serialised: compare shares, not absolutes)
# 2. one --set full capture of each window kernel of interest
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --profile-steps 0 --no-cpu-baseline --secondary="
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $CMD > $OUT/${TAG}_launches.log 2>&1
for k in "tc_gemm2_kernel:4" "rec_persist_kernel:2" "k_rms:4" "k_pfac_rows:1" "k_embed:2"; do
  name=${k%%:*}; cnt=${k##*:}
  ncu --set full --clock-control none --import-source on -k regex:$name -s $((cnt * 3)) -c $cnt \
      -o $OUT/${TAG}_prof_${name} $CMD > $OUT/${TAG}_prof_${name}.log 2>&1
done
# the fp32-class tensor-core mode's GEMM (3xTF32) at C2
ncu --set full --clock-control none --import-source on -k regex:tc_tf32x3 -s 0 -c 40 \
    -o $OUT/${TAG}_prof_tc_tf32x3 python bench.py --steps 2 --warmup 2 --no-e2e --profile-steps 0 \
    --no-cpu-baseline --secondary= --config c2 --precision tf32x3 > $OUT/${TAG}_prof_tc_tf32x3.log 2>&1
ls -la $OUT
