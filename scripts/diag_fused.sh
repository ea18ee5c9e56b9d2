# Tuning diagnostics: bench_quick over the variants/ builds (scripts/build_variant.sh)
for v in base $(ls variants); do
  if [ $v = base ]; then unset DL_LIB_PATH; else export DL_LIB_PATH=variants/$v/libdesklm_cuda.so; fi
  echo "== $v"
  python scripts/bench_quick.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --secondary ""
done
