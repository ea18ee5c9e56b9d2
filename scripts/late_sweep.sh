# Tuning: fused dW_out update vs the late fork (bf16 dW_out + the dense
# update on the side stream under the backward recurrence) at C3
Q="python scripts/bench_quick.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --secondary="
echo "== fused"; $Q
echo "== late b1"; DL_FUSE_OUT=0 DL_FORK_LATE=1 DL_RMS_G16_BLOCKS=1 $Q
echo "== late b2"; DL_FUSE_OUT=0 DL_FORK_LATE=1 DL_RMS_G16_BLOCKS=2 $Q
echo "== late b4"; DL_FUSE_OUT=0 DL_FORK_LATE=1 DL_RMS_G16_BLOCKS=4 $Q
echo "== unfused serial b4"; DL_FUSE_OUT=0 DL_RMS_G16_BLOCKS=4 $Q
