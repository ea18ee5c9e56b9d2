#!/bin/bash
# launch list per variants/<name> build, filtered by a kernel-name regex
PAT=${1:-.}
for d in variants/*/; do
  n=$(basename $d)
  echo "== $n"
  DL_LIB_PATH=$PWD/variants/$n/libdesklm_cuda.so bash scripts/launches.sh v_$n | grep -E "$PAT|total"
done
