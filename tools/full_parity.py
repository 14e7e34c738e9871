"""Development aid: every instance of a configuration vs the oracle (per-instance bar of
tests/parity.py without the conditioning fallback).  usage: full_parity.py CFG SEED [LIB]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2109_13030_b200 import bmc
if len(sys.argv) > 3:
    bmc.load_library(os.path.abspath(sys.argv[3]))
from paper_2109_13030_b200 import solver_for
from synth import CONFIGS, make_problem
from oracle import Oracle
from tests.helpers import oracle_params, bpoly_basis
from tests.parity import _deviations, _fails
cfg = CONFIGS[sys.argv[1]]; pr = make_problem(cfg, int(sys.argv[2]))
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
g = solver_for(cfg, device=0).solve(d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], cfg.K)
torch.cuda.synchronize(); g = {k: v.cpu().numpy() for k, v in g.items()}
ref = Oracle(oracle_params(cfg), cfg.n).solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K)
P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
dt, dJ, dr = _deviations(P, g["coeffs"], ref["coeffs"], g["cost"], ref["cost"], g["residual"], ref["residual"])
bad = _fails(cfg, dt, dJ, dr, ref["cost"], ref["residual"])
rel = dJ / np.abs(ref["cost"])
print(f"{os.path.basename(sys.argv[3]) if len(sys.argv) > 3 else 'libbmc.so'} {cfg.name} seed {sys.argv[2]}: "
      f"{bad.sum()} / {len(bad)} miss the bar; max dtraj {dt.max():.2e}, max rel dJ {rel.max():.2e}, "
      f"p99 dtraj {np.percentile(dt, 99):.2e}; failing {np.where(bad)[0][:10].tolist()}; "
      f"best gpu {int(g['best'][0])} oracle {ref['best_index']}")
