# diagnostics: narrow-TSQR kernels (thread / lane-group streams, the default
# for m <= 32) against warp streams (TTSVD_TSQR=ws)
for sel in "" ws; do
  echo "== ${sel:-default}"
  TTSVD_TSQR=$sel python tools/tsqr_shapes.py 268435456x4 134217728x8 16777216x12 16777216x16 67108864x16 8388608x24 33554432x32
done
