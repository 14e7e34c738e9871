#!/bin/bash
# bitwise comparison of the current build against tools/prev/libbmc_prev.so + timings
OUT=gpurun_out/${1:-cmp}; mkdir -p $OUT
for c in "C1 8" "C2 100" "C3 1000" "C4 1000" "C5 2000"; do
  set -- $c
  timeout 300 python tools/cmp_prev.py tools/prev/libbmc_prev.so $1 $2 $OUT/prev_$1.npz
  timeout 300 python tools/cmp_prev.py paper_2109_13030_b200/libbmc.so $1 $2 $OUT/new_$1.npz
  python - $OUT $1 <<'PY'
import sys, numpy as np
o, c = sys.argv[1], sys.argv[2]
a, b = np.load(f"{o}/prev_{c}.npz"), np.load(f"{o}/new_{c}.npz")
for k in a.files:
    same = np.array_equal(a[k], b[k], equal_nan=True) if a[k].dtype.kind == 'f' else np.array_equal(a[k], b[k])
    diff = 0 if same else np.nanmax(np.abs(a[k].astype(np.float64) - b[k].astype(np.float64)))
    print(c, k, "bitwise" if same else f"DIFF max {diff:.3g} n={np.sum(a[k]!=b[k])}")
PY
done
