"""Development aid: one configuration's instances vs the oracle for several team sizes / libs.
usage: python tools/inst_check.py CFG SEED B [LIB...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import CONFIGS, make_problem
from oracle import Oracle
from tests.helpers import oracle_params, bpoly_basis
cfg = CONFIGS[sys.argv[1]]; seed = int(sys.argv[2]); B = int(sys.argv[3])
pr = make_problem(cfg, seed, B=B)
ref = Oracle(oracle_params(cfg), cfg.n).solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K)
P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
libs = sys.argv[4:] or ["paper_2109_13030_b200/libbmc.so"]
import subprocess, json
for lib in libs:
    for team in (1, 2, 4):
        code = f'''
import sys, os, numpy as np, torch
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
from paper_2109_13030_b200 import bmc, solver_for
bmc.load_library(os.path.abspath({lib!r}))
from synth import CONFIGS, make_problem
cfg = CONFIGS[{sys.argv[1]!r}]; pr = make_problem(cfg, {seed}, B={B})
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
o = solver_for(cfg, device=0).solve(d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], cfg.K)
torch.cuda.synchronize()
np.save("/tmp/inst_c.npy", o["coeffs"].cpu().numpy()); np.save("/tmp/inst_j.npy", o["cost"].cpu().numpy())
'''
        env = dict(os.environ, BMC_TEAM=str(team))
        subprocess.run([sys.executable, "-c", code], env=env, check=True, capture_output=True)
        c = np.load("/tmp/inst_c.npy").astype(np.float64); J = np.load("/tmp/inst_j.npy")
        dt = np.maximum(np.abs((c[:, 0] - ref["coeffs"][:, 0]) @ P.T).max(1), np.abs((c[:, 2] - ref["coeffs"][:, 2]) @ P.T).max(1))
        dj = np.abs(J - ref["cost"]) / np.abs(ref["cost"])
        worst = np.argsort(-dt)[:3]
        print(f"{os.path.basename(lib)} T={team}: max dtraj {dt.max():.2e} worst {worst.tolist()} {dt[worst]} max rel dJ {dj.max():.2e}")
