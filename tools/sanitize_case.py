"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every team size (1, 2 with the round-0 hand-off, 4), circular and elliptical
obstacles, a ragged tail, the exchange kernels and the STOMP sampler.
usage: compute-sanitizer --tool T python tools/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2109_13030_b200 import solver_for
from synth import CONFIGS, make_problem

torch.cuda.set_device(0)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
K = int(os.environ.get("SAN_K", "4"))
cases = [("C1", None, {}), ("C3", 300, {"BMC_TEAM": "2"}), ("C3", 150, {"BMC_TEAM": "1"}),
         ("C2", 37, {"BMC_TEAM": "4"}), ("C4", 149, {})]
for name, B, env in cases:
    os.environ.pop("BMC_TEAM", None)
    os.environ.update(env)
    cfg = CONFIGS[name] if B is None else CONFIGS[name].with_(B=B)
    pr = make_problem(cfg, 1)
    s = solver_for(cfg, device=0)
    out = s.solve(d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], K, trace=True)
    torch.cuda.synchronize()
    print(name, B, env, "best", int(out["best"][0].item()), flush=True)
# ellipses (general collision loop, scaled rule)
cfg = CONFIGS["C2"].with_(B=20, n=6)
pr = make_problem(cfg, 2)
pr["obs_ab"] = np.stack([np.linspace(0.5, 1.1, 6), np.linspace(0.9, 0.4, 6)], 1).astype(np.float32)
s = solver_for(cfg, device=0, alpha_rule=1)
out = s.solve(d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], K)
torch.cuda.synchronize()
print("ellipse best", int(out["best"][0].item()))
# host path (page-locked zero-copy and pageable staging), sampler, exchange kernels
h = s.solve_host(pr["init"], pr["obs_xy"], pr["obs_ab"], pr["bnd"], K)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
h2 = s.solve_host(pin(pr["init"]), pin(pr["obs_xy"]), pin(pr["obs_ab"]), pr["bnd"], K)
assert np.array_equal(h["coeffs"], h2["coeffs"])
smp = s.sample_init(257, pr["bnd"], seed=7)
torch.cuda.synchronize()
from paper_2109_13030_b200.distributed import RECORD_WORDS  # noqa: E402
import ctypes as C  # noqa: E402
from paper_2109_13030_b200.bmc import load_library  # noqa: E402
L = load_library()
rec = torch.zeros(2 * RECORD_WORDS, dtype=torch.int64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
L.bmc_pack_best(C.c_void_p(out["best"].data_ptr()), C.c_void_p(out["coeffs"].data_ptr()), C.c_int64(0),
                C.c_void_p(rec.data_ptr()), st)
L.bmc_pack_best(C.c_void_p(out["best"].data_ptr()), C.c_void_p(out["coeffs"].data_ptr()), C.c_int64(0),
                C.c_void_p(rec[RECORD_WORDS:].data_ptr()), st)
best = torch.zeros(2, dtype=torch.int64, device="cuda")
co = torch.zeros(55, dtype=torch.float32, device="cuda")
L.bmc_select_best(C.c_void_p(rec.data_ptr()), C.c_int32(2), C.c_void_p(best.data_ptr()), C.c_void_p(co.data_ptr()), st)
torch.cuda.synchronize()
print("sanitize cases done")
