"""Quick GPU probe: parity stats + timing on C1..C4 (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import Oracle
from synth import CONFIGS, make_problem
from tests.helpers import oracle_params, bpoly_basis
from paper_2109_13030_b200 import solver_for

torch.cuda.set_device(0)
def dev(a): return torch.from_numpy(np.ascontiguousarray(a)).cuda()

def timeit(cfg, pr, reps=5):
    s = solver_for(cfg, device=0)
    args = (dev(pr["init"]), dev(pr["obs_xy"]), dev(pr["obs_ab"]), pr["bnd"], cfg.K)
    out = s.solve(*args); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); s.solve(*args, out=out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return out, min(ts), float(np.median(ts))

for name, B_or in [("C1", None), ("C2", None), ("C3", None), ("C4", None)]:
    cfg = CONFIGS[name]
    pr = make_problem(cfg, 0)
    out, tmin, tmed = timeit(cfg, pr)
    g = {k: v.cpu().numpy() for k, v in out.items()}
    nsamp = min(cfg.B, 12)
    idx = np.arange(nsamp)
    sub = dict(pr); sub["init"] = pr["init"][idx]
    o = Oracle(oracle_params(cfg), cfg.n)
    t0 = time.time(); r = o.solve(sub["bnd"], sub["obs_xy"], sub["obs_ab"], sub["init"], cfg.K); tcpu = time.time() - t0
    P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    cg = g["coeffs"][idx].astype(np.float64); cr = r["coeffs"]
    dtraj = np.maximum(np.abs((cg[:, 0] - cr[:, 0]) @ P.T).max(1), np.abs((cg[:, 2] - cr[:, 2]) @ P.T).max(1))
    dJ = np.abs(g["cost"][idx] - r["cost"]) / (np.abs(r["cost"]) + 1e-12)
    dr = np.abs(g["residual"][idx] - r["residual"])
    print(f"{name}: B={cfg.B} K={cfg.K} gpu {tmin:.3f} ms (med {tmed:.3f}); traj.iter/s {cfg.B*cfg.K/tmin*1e3:.3e}; "
          f"oracle {nsamp} inst {tcpu:.2f}s")
    print(f"   dtraj per inst: {np.array2string(dtraj, precision=2)}")
    print(f"   rel dJ max {dJ.max():.2e}  dr max {dr.max():.2e}  r1 gpu {np.array2string(g['residual'][idx,0], precision=3)}")
    print(f"   r1 ref {np.array2string(r['residual'][:,0], precision=3)}")
    print(f"   best gpu {int(g['best'][0])}")
