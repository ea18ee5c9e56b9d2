#!/bin/bash
# Tuning experiments only: build libdesklm_cuda.so with extra nvcc flags into
# variants/<name>/ (select it at run time with DL_LIB_PATH=variants/<name>/libdesklm_cuda.so).
#   scripts/build_variant.sh <name> [-DFOO=1 ...]
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/variants/$NAME
mkdir -p $OUT
cd $ROOT/paper_1502_00512_b200
FL="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -ccbin /usr/bin/g++ --expt-relaxed-constexpr $*"
objs=""
for s in csrc/*.cu; do
  o=$OUT/$(basename $s .cu).o
  /usr/local/cuda/bin/nvcc $FL -c $s -o $o &
  objs="$objs $o"
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o $OUT/libdesklm_cuda.so $objs -lnccl
rm -f $OUT/*.o
echo built $OUT/libdesklm_cuda.so
