#!/bin/bash
# fixed cost of a solve (development aid): back-to-back GPU time at K = 0, 1, 100 for
# the libraries given, then the PROFILE build's per-CTA wall-clock split at K = 0 and 100
for lib in "$@"; do echo "== $lib"; BMC_LIB=paper_2109_13030_b200/$lib python tools/timek.py C3 0 1 100 | grep "back to back"; done
cp paper_2109_13030_b200/libbmc.so /tmp/keep.so; cp paper_2109_13030_b200/${PROFLIB:-libbmc_prof.so} paper_2109_13030_b200/libbmc.so
for K in 0 100; do BMC_PROF=1 python - $K <<'PY' 2>&1 | grep "CTA wall" | tail -1
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from synth import CONFIGS, make_problem
from paper_2109_13030_b200 import solver_for
K = int(sys.argv[1]); cfg = CONFIGS["C3"]; pr = make_problem(cfg, 0)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
s = solver_for(cfg, device=0)
for _ in range(3):
    s.solve(d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], K); torch.cuda.synchronize()
PY
done
cp /tmp/keep.so paper_2109_13030_b200/libbmc.so
