"""r1 traces of chosen instances, GPU (full-batch launch) vs oracle (development aid):
python tools/inst_trace.py CFG SEED INST [INST ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2109_13030_b200 import solver_for
from synth import CONFIGS, make_problem
from oracle import Oracle
from tests.helpers import oracle_params
cfg = CONFIGS[sys.argv[1]]; pr = make_problem(cfg, int(sys.argv[2])); idx = [int(x) for x in sys.argv[3:]]
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
g = solver_for(cfg, device=0).solve(d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], cfg.K, trace=True)
torch.cuda.synchronize()
gt = g["res_trace"].cpu().numpy()[idx]
sub = dict(pr); sub["init"] = pr["init"][idx]
o = Oracle(oracle_params(cfg), cfg.n).solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], sub["init"], cfg.K, trace=True)
ot = o["res_trace"]
for j, i in enumerate(idx):
    rel = np.abs(gt[j] - ot[j]) / np.maximum(ot[j], 1e-6)
    first = [k for k in range(cfg.K) if rel[k] > 1e-3]
    print(f"inst {i}: first iteration with |dr1|/r1 > 1e-3: {first[0] if first else None}; "
          f"rel dr1 at k = 10, 50, 100, 150, {cfg.K - 1}: " +
          " ".join(f"{rel[min(k, cfg.K - 1)]:.1e}" for k in (10, 50, 100, 150, cfg.K - 1)))
    print("   r1 oracle (every 20th):", " ".join(f"{x:.4f}" for x in ot[j][::20]))
