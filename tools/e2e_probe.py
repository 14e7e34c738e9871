"""Where the end-to-end time of bmc_solve_host goes (dev aid): wall time per call at
K = 0 and K = 100 through the host path (pinned, mapped in place), the device path
with a synchronize, and the cost of one cudaPointerGetAttributes query."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import CONFIGS, make_problem
from paper_2109_13030_b200 import solver_for

cfg = CONFIGS["C3"]; pr = make_problem(cfg, 0)
s = solver_for(cfg, device=0)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
hi, ho, ha = pin(pr["init"]), pin(pr["obs_xy"]), pin(pr["obs_ab"])
B = cfg.B
out = dict(coeffs=pin(np.empty((B, 5, 11), np.float32)), lambda_out=pin(np.empty((B, 5, 11), np.float32)),
           residual=pin(np.empty((B, 2), np.float32)), cost=pin(np.empty((B,), np.float32)), best=pin(np.empty(2, np.int64)))
out_nl = {k: v for k, v in out.items() if k != "lambda_out"}
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
di, do, da = d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"])
def wall(f, n=50):
    for _ in range(5): f()
    t = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t) / n * 1e6
for K in (0, 100):
    print(f"K={K}: host path {wall(lambda: s.solve_host(hi, ho, ha, pr['bnd'], K, out=out)):.1f} us, "
          f"host path without lambda_out {wall(lambda: s.solve_host(hi, ho, ha, pr['bnd'], K, out=out_nl)):.1f} us, "
          f"device path + sync {wall(lambda: (s.solve(di, do, da, pr['bnd'], K), torch.cuda.synchronize())):.1f} us")
rt = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if rt is not None:
    attr = (C.c_byte * 64)()
    p = C.c_void_p(out["coeffs"].ctypes.data)
    t = time.perf_counter()
    for _ in range(1000): rt.cudaPointerGetAttributes(attr, p)
    print(f"cudaPointerGetAttributes: {(time.perf_counter() - t) * 1e3:.2f} us per call")
