# diagnostics: block-Jacobi variants (diagnostics builds under tools/_var)
for lib in "" $BJ_LIBS; do
  echo "#### ${lib:-default}"
  TTSVD_LIB_VARIANT=$lib python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); p=d['phases_ms']; print(d['value'], p['small_svd'], p['svd_sweeps'])"
done
