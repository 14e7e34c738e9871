"""Development aid: run one configuration with a given libbmc.so and save the
outputs, so two builds can be compared bit for bit.
usage: python tools/cmp_prev.py LIB CFG B OUT.npz"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2109_13030_b200 import bmc
bmc.load_library(os.path.abspath(sys.argv[1]))
from synth import CONFIGS, make_problem
from paper_2109_13030_b200 import solver_for
torch.cuda.set_device(0)
cfg = CONFIGS[sys.argv[2]].with_(B=int(sys.argv[3]))
pr = make_problem(cfg, 0)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
s = solver_for(cfg, device=0)
out = s.solve(d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], cfg.K)
torch.cuda.synchronize()
np.savez(sys.argv[4], **{k: v.cpu().numpy() for k, v in out.items()})
