"""Time one configuration at several iteration counts (development aid):
python tools/timek.py C3 0 1 10 100 -> fixed cost (prologue, init iteration, epilogue) and per-iteration slope"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import CONFIGS, make_problem
from paper_2109_13030_b200 import solver_for, bmc
if os.environ.get("BMC_LIB"):   # experiments: a variant build (make TAG=...)
    bmc.load_library(os.path.abspath(os.environ["BMC_LIB"]))
torch.cuda.set_device(0)
cfg = CONFIGS[sys.argv[1]]
pr = make_problem(cfg, 0)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
s = solver_for(cfg, device=0)
args = (d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"])
for K in map(int, sys.argv[2:]):
    out = s.solve(*args, K)
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); s.solve(*args, K, out=out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{cfg.name} K={K}: {np.median(ts) * 1e3:.1f} us (min {min(ts) * 1e3:.1f})")
# back-to-back launches between one pair of events: GPU time per solve without host gaps
for K in map(int, sys.argv[2:]):
    out = s.solve(*args, K)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        s.solve(*args, K, out=out)
    e1.record(); torch.cuda.synchronize()
    print(f"{cfg.name} K={K}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per solve, 50 back to back")
