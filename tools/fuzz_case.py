"""Re-run one case of tests/test_gpu_fuzz.py with overrides and print the parity
stats instead of asserting (dev aid):
  python tools/fuzz_case.py SEED [key=value ...]   keys: team, mask, ell (0/1), rule, m_sym (1: symmetric r), K, lib"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import Oracle
from synth import make_problem
from tests.helpers import oracle_params
from tests.parity import compare
from tests.test_gpu_fuzz import _case
from paper_2109_13030_b200 import bmc, solver_for

seed = int(sys.argv[1]); ov = dict(a.split("=") for a in sys.argv[2:])
if "lib" in ov:
    bmc.load_library(os.path.abspath(ov["lib"]))
cfg, kw, ellipses, team, warm, rng = _case(seed)
pr = make_problem(cfg, 30 + seed)
if ellipses:
    pr["obs_ab"] = np.stack([rng.uniform(0.4, 0.9, cfg.n), rng.uniform(0.3, 0.8, cfg.n)], 1).astype(np.float32)
if "team" in ov: team = int(ov["team"])
if "mask" in ov: kw["boundary_mask"] = int(ov["mask"], 0)
if "rule" in ov: kw["alpha_rule"] = int(ov["rule"])
if "m_sym" in ov:
    m = cfg.m; kw["r"] = list(np.round(np.linspace(-0.3 * (m - 1), 0.3 * (m - 1), m), 6))
if "K" in ov: cfg = cfg.with_(K=int(ov["K"]))
if ov.get("ell") == "0" and cfg.n:
    pr["obs_ab"] = np.repeat(pr["obs_ab"][:, :1], 2, axis=1).copy()
print("case", seed, dict(q=cfg.q, m=cfg.m, n=cfg.n, B=cfg.B, K=cfg.K), kw, "team", team, "warm", warm)
o = Oracle(oracle_params(cfg, **kw), cfg.n)
s = solver_for(cfg, device=0, **kw)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
lam = o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], 5)["lambda_out"].astype(np.float32) if warm else None
out = s.solve(d(pr["init"]), d(pr["obs_xy"]) if cfg.n else None, d(pr["obs_ab"]) if cfg.n else None, pr["bnd"],
              cfg.K, lambda_in=None if lam is None else d(lam), team=team)
torch.cuda.synchronize()
g = {k: v.cpu().numpy() for k, v in out.items()}
r = o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K, lambda_in=lam)
try:
    st = compare(cfg, g, r, cfg.res_tol, "case", oracle=o, problem=pr, lambda_in=lam)
    print("PASS", {k: v for k, v in st.items() if k.startswith("max_d")}, "accepted", len(st["fp32_model_accepted"]))
except AssertionError as e:
    msg = str(e)
    print("FAIL", msg[msg.find("'max_dtraj'"):msg.find("'fp32_model_accepted'")], msg[msg.find("failing instances"):])
J = np.asarray(r["cost"]); dJ = np.abs(g["cost"] - J) / np.abs(J)
print("rel dJ: median %.2e p90 %.2e max %.2e" % (np.median(dJ), np.percentile(dJ, 90), dJ.max()))
lg = np.asarray(g["lambda_out"], np.float64).reshape(len(J), -1); lr = np.asarray(r["lambda_out"]).reshape(len(J), -1)
dl = np.abs(lg - lr).max(1); worst = int(dl.argmax())
print("lambda: worst inst %d dlam %.2e max|lam| %.2e; worst entry %d (channel block %d)" %
      (worst, dl[worst], np.abs(lr[worst]).max(), int(np.abs(lg[worst] - lr[worst]).argmax()),
       int(np.abs(lg[worst] - lr[worst]).argmax()) // 11))
