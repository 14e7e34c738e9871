#!/bin/bash
# per-phase cycles of the PROFILE build (development aid): CFG=C3 tools/prof_c.sh [lib]
LIB=${1:-libbmc_prof.so}
BMC_PROF=1 BMC_LIB=paper_2109_13030_b200/$LIB python - ${CFG:-C3} <<'PY' 2>&1 | grep "bmc prof" | tail -8
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from synth import CONFIGS, make_problem
import os
from paper_2109_13030_b200 import bmc, solver_for
bmc.load_library(os.path.abspath(os.environ["BMC_LIB"]))
cfg = CONFIGS[sys.argv[1]]; pr = make_problem(cfg, 0)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
s = solver_for(cfg, device=0)
for _ in range(2):
    s.solve(d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], cfg.K); torch.cuda.synchronize()
PY
