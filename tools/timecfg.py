"""Time one configuration (development aid): python tools/timecfg.py C3 [B]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import CONFIGS, make_problem
from paper_2109_13030_b200 import solver_for, bmc
if os.environ.get("BMC_LIB"):   # experiments: a variant build (make TAG=...)
    bmc.load_library(os.path.abspath(os.environ["BMC_LIB"]))
torch.cuda.set_device(0)
cfg = CONFIGS[sys.argv[1]]
if len(sys.argv) > 2: cfg = cfg.with_(B=int(sys.argv[2]))
pr = make_problem(cfg, 0)
kw = {}
if os.environ.get("BMC_ELL"):   # ellipse scene (NEXT-4): a ~ U(0.5, 0.9), b ~ U(0.35, 0.7), alpha_rule = BMC_ELL
    rng = np.random.default_rng(1000)
    pr["obs_ab"] = np.stack([rng.uniform(0.5, 0.9, cfg.n), rng.uniform(0.35, 0.7, cfg.n)], 1).astype(np.float32)
    kw["alpha_rule"] = int(os.environ["BMC_ELL"])
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
s = solver_for(cfg, device=0, **kw)
args = (d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], cfg.K)
out = s.solve(*args); torch.cuda.synchronize()
ref = {k: v.clone() for k, v in out.items()}
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); s.solve(*args, out=out); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{os.environ.get('BMC_LIB', '')} {cfg.name}{' ell' + os.environ['BMC_ELL'] if os.environ.get('BMC_ELL') else ''} B={cfg.B} wmax={os.environ.get('BMC_WMAX', '-')} team={os.environ.get('BMC_TEAM','1')} ipc={os.environ.get('BMC_IPC','-')}: "
      f"{min(ts):.3f} ms (med {np.median(ts):.3f})  best={int(out['best'][0])}  cost0={float(out['cost'][0]):.6f}")
