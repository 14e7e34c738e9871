"""Every instance of a configuration vs the oracle with the full parity harness
(tests/parity.compare: the per-instance bar plus the conditioning fallback).
usage: full_compare.py CFG SEED  -> accepted-as-ill-conditioned list or the failure"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2109_13030_b200 import solver_for
from synth import CONFIGS, make_problem
from oracle import Oracle
from tests.helpers import oracle_params
from tests.parity import compare
cfg = CONFIGS[sys.argv[1]]; pr = make_problem(cfg, int(sys.argv[2]))
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
g = solver_for(cfg, device=0).solve(d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], cfg.K)
torch.cuda.synchronize(); g = {k: v.cpu().numpy() for k, v in g.items()}
o = Oracle(oracle_params(cfg), cfg.n)
ref = o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K)
try:
    st = compare(cfg, g, ref, cfg.res_tol, f"{cfg.name} seed {sys.argv[2]} all", oracle=o, problem=pr)
    ill = st["ill_conditioned"]
    print(f"{cfg.name} seed {sys.argv[2]}: PASS, {len(ill)} accepted as ill-conditioned; "
          f"max dtraj {st['max_dtraj']:.2e}; worst ratio dtraj/spread "
          f"{max([x['dtraj'] / max(x['spread_traj'], 1e-12) for x in ill] or [0]):.2f}")
except AssertionError as e:
    msg = str(e); print(f"{cfg.name} seed {sys.argv[2]}: FAIL ... {msg[msg.index("failing instances"):] if "failing instances" in msg else msg[-400:]}")
    # detail of the rejected instances: deviation vs the oracle's own spread
    from tests.parity import _deviations, _fails, intrinsic_spread
    from tests.helpers import bpoly_basis
    P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    dt, dJ, dr = _deviations(P, g["coeffs"], ref["coeffs"], g["cost"], ref["cost"], g["residual"], ref["residual"])
    bad = np.where(_fails(cfg, dt, dJ, dr, ref["cost"], ref["residual"]))[0]
    s_t, s_J, s_r = intrinsic_spread(cfg, o, pr, bad, cfg.K)
    for b, a1, a2, a3, b1, b2, b3 in zip(bad, dt[bad], dJ[bad], dr[bad].max(1), s_t, s_J, s_r.max(1)):
        flag = "" if (a1 <= max(1e-3, 10 * b1) and a2 <= max(1e-4 * abs(ref["cost"][b]) + 1e-6, 10 * b2)
                      and a3 <= max(1e-4 * ref["residual"][b].max() + 2e-5, 10 * b3)) else "  <-- rejected"
        print(f"  inst {b}: dtraj {a1:.2e} (spread {b1:.2e})  dJ {a2:.2e} (spread {b2:.2e}, J {ref['cost'][b]:.3e})"
              f"  dr {a3:.2e} (spread {b3:.2e}){flag}")
