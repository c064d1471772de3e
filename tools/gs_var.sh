# diagnostics: time TSQR variants (TTSVD_GS selects the group-stream shape,
# TTSVD_LIB_VARIANT a diagnostics build of the library)
for lib in "" $GS_LIBS; do
  echo "#### lib ${lib:-default}"
  for v in 16,2,8 16,4,8; do echo "== $v"; TTSVD_LIB_VARIANT=$lib TTSVD_GS=$v python tools/tsqr_shapes.py 16777216x16 67108864x16; done
  for v in 32,8,8; do echo "== $v"; TTSVD_LIB_VARIANT=$lib TTSVD_GS=$v python tools/tsqr_shapes.py 33554432x32 8388608x24; done
  echo "== pt"; TTSVD_LIB_VARIANT=$lib python tools/tsqr_shapes.py 134217728x8 153391689x7 268435456x4
done
