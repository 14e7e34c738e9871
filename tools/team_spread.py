"""Rounding-noise floor of sensitive instances: the same full-batch solve with
different team sizes (different fp32 summation orders) vs the oracle
(development aid): python tools/team_spread.py CFG SEED INST [INST ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2109_13030_b200 import solver_for
from synth import CONFIGS, make_problem
from oracle import Oracle
from tests.helpers import oracle_params, bpoly_basis
from tests.parity import _deviations
cfg = CONFIGS[sys.argv[1]]; pr = make_problem(cfg, int(sys.argv[2])); idx = [int(x) for x in sys.argv[3:]]
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
res = {}
for team in ("2", "1", "4"):
    os.environ["BMC_TEAM"] = team
    g = solver_for(cfg, device=0).solve(d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], cfg.K)
    torch.cuda.synchronize()
    res[team] = {k: v.cpu().numpy()[idx] for k, v in g.items() if k != "best"}
sub = dict(pr); sub["init"] = pr["init"][idx]
o = Oracle(oracle_params(cfg), cfg.n).solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], sub["init"], cfg.K)
P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
def dev(a, b):
    return _deviations(P, a["coeffs"], b["coeffs"], a["cost"], b["cost"], a["residual"], b["residual"])
for lab, (a, b) in {"T2 vs oracle": (res["2"], o), "T1 vs oracle": (res["1"], o), "T4 vs oracle": (res["4"], o),
                    "T2 vs T1": (res["2"], res["1"]), "T2 vs T4": (res["2"], res["4"])}.items():
    dt, dJ, dr = dev(a, b)
    print(f"{lab:14s} dtraj " + " ".join(f"{x:.1e}" for x in dt) + " | rel dJ " +
          " ".join(f"{x:.1e}" for x in dJ / np.abs(o["cost"])))
