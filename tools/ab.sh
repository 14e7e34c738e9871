#!/bin/bash
# A/B timing of library variants (development aid): tools/ab.sh TAG lib1 lib2 ...
TAG=$1; shift; LOG=gpurun_out/$TAG.log; mkdir -p gpurun_out/$TAG; : > $LOG
for lib in "$@"; do
  for c in "C3" "C4" "C5" "C3 148"; do BMC_LIB=paper_2109_13030_b200/$lib timeout -s KILL 120 python tools/timecfg.py $c 2>&1 | grep -E "^ C|^paper" ; done >> $LOG
  for c in C1 C2 C3 C4; do
    timeout -s KILL 120 python tools/cmp_prev.py paper_2109_13030_b200/$lib $c 1000 gpurun_out/$TAG/${lib}_$c.npz > /dev/null 2>&1
  done
done
python - "$TAG" "$@" >> $LOG <<'PY'
import sys, numpy as np
tag, libs = sys.argv[1], sys.argv[2:]
for lib in libs[1:]:
    for c in ("C1", "C2", "C3", "C4"):
        a, b = np.load(f"gpurun_out/{tag}/{libs[0]}_{c}.npz"), np.load(f"gpurun_out/{tag}/{lib}_{c}.npz")
        bad = [k for k in a.files if not np.array_equal(a[k], b[k], equal_nan=True)]
        print(lib, c, "bitwise" if not bad else "DIFF " + " ".join(f"{k}:{np.nanmax(np.abs(a[k].astype(float)-b[k].astype(float))):.2g}" for k in bad))
PY
cat $LOG
