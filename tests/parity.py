"""GPU <-> oracle comparison used by the -m gpu tests and smoke().

The bar (BASELINE.json north_star), per instance:
  * trajectory x, y: max over t of |P (c_gpu - c_oracle)| <= TRAJ_TOL = 1e-3 m,
    with P the fp64 basis (scipy BPoly, independent of both sides);
  * heading psi and the copies c, s (the rest of the trajectory):
    <= ANGLE_TOL = 1e-3 rad (dimensionless for c, s) -- reading P1 of DESIGN.md:
    1e-3 rad moves a circle centre (|r_i| <= 0.75 m) by < 1e-3 m;
  * cost J: |dJ| <= 1e-4 |J| + 1e-8 q;
  * residuals r1, r_psi: |dr| <= 1e-4 |r| + RES_FLOOR, RES_FLOOR = 2e-5: the GPU
    evaluates the per-row residuals in fp32, so each row carries ~1e-7 absolute
    rounding and ||.||_2 over ~1e4 rows an absolute floor of ~1e-5;
  * multipliers lambda_out: max |d lambda| <= 1e-4 max|lambda| + LAM_FLOOR (the
    north star's relative 1e-4, norm-wise: the entries differ by orders of
    magnitude); LAM_FLOOR = rho K sqrt(q) 3e-7 is K multiplier steps of a
    contraction over q samples of fp32 residuals (~3e-7 absolute each);
  * best index identical, unless the scene is ambiguous (a residual within 1e-3
    relative of tau, or the oracle's best and runner-up keys within 1e-3
    relative): then the oracle's value at the GPU's pick must be within 1e-4 of
    the oracle's best value.

fp32 rounding model: the AM map is non-smooth and
non-convex; on some instances it amplifies perturbations by >1e3 over 100
iterations, so fp32 rounding ALONE moves the answer by more than the bar and no
fp32 implementation can meet it there.  For an instance that misses the bar, the
oracle is re-run N_MODEL times with its fp32 rounding model (oracle.h
`fp32_model`: every quantity the product path holds in fp32 rounded where it is
formed, stochastically, one seed per run); the instance passes only if, for
every quantity that misses the bar, the GPU deviation is within KAPPA times the
largest deviation of those runs from the fp64 oracle.  KAPPA is calibrated on
the oracle alone (tools/calibrate_kappa.py): further model runs standing in
for "another fp32 implementation" stay within KAPPA x the N_MODEL-run spread on
every calibration instance.  A well-conditioned instance (model spread ~1e-6)
gets no slack.  Every such acceptance is reported.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from tests.helpers import bpoly_basis

TRAJ_TOL = 1e-3
ANGLE_TOL = 1e-3
COST_RTOL = 1e-4
RES_RTOL = 1e-4
RES_FLOOR = 2e-5
LAM_RTOL = 1e-4
LAM_UNIT = 3e-7          # absolute fp32 rounding of one residual sample (LAM_FLOOR)
N_MODEL = 4              # fp32-model runs per failing instance
MODEL_SEED0 = 1          # their seeds: MODEL_SEED0 .. MODEL_SEED0 + N_MODEL - 1
KAPPA = 8.0              # tools/calibrate_kappa.py (profiles/kappa_calibration.json): over 423 probe
                         # misses of the bar (C2-C4) the probe/spread ratio has median 0.90, p99 3.1,
                         # max 7.6 -- another fp32 implementation can land that far on a chaotic orbit

QUANTITIES = ("traj", "psi", "copy", "cost", "r1", "rpsi", "lam")


def key_value(r1, J, tau):
    feas = r1 <= tau
    v = np.where(feas, J, r1).astype(np.float32)
    return feas, v


def deviations(P, g: dict, r: dict) -> dict:
    """Per-instance deviation of each quantity between two result sets."""
    cg = np.asarray(g["coeffs"], np.float64)
    cr = np.asarray(r["coeffs"], np.float64)
    ev = lambda blk: np.max(np.abs((cg[:, blk] - cr[:, blk]) @ P.T), axis=1)
    rg = np.asarray(g["residual"], np.float64)
    rr = np.asarray(r["residual"], np.float64)
    d = dict(traj=np.maximum(ev(0), ev(2)), psi=ev(4), copy=np.maximum(ev(1), ev(3)),
             cost=np.abs(np.asarray(g["cost"], np.float64) - np.asarray(r["cost"], np.float64)),
             r1=np.abs(rg[:, 0] - rr[:, 0]), rpsi=np.abs(rg[:, 1] - rr[:, 1]))
    if "lambda_out" in g and "lambda_out" in r:
        lg = np.asarray(g["lambda_out"], np.float64).reshape(len(cg), -1)
        lr = np.asarray(r["lambda_out"], np.float64).reshape(len(cg), -1)
        d["lam"] = np.max(np.abs(lg - lr), axis=1)
    return d


def bars(cfg, r: dict, iters: int) -> dict:
    """Per-instance tolerance of each quantity (module docstring)."""
    J = np.abs(np.asarray(r["cost"], np.float64))
    rr = np.abs(np.asarray(r["residual"], np.float64))
    n = len(J)
    b = dict(traj=np.full(n, TRAJ_TOL), psi=np.full(n, ANGLE_TOL), copy=np.full(n, ANGLE_TOL),
             cost=COST_RTOL * J + 1e-8 * cfg.q, r1=RES_RTOL * rr[:, 0] + RES_FLOOR,
             rpsi=RES_RTOL * rr[:, 1] + RES_FLOOR)
    if "lambda_out" in r:
        lam = np.abs(np.asarray(r["lambda_out"], np.float64)).reshape(n, -1).max(axis=1)
        b["lam"] = LAM_RTOL * lam + cfg.rho * max(iters, 1) * np.sqrt(cfg.q) * LAM_UNIT
    return b


def fp32_spread(oracle, problem, rows, iters, ref_rows: dict, lambda_in=None, P=None,
                seeds=None) -> dict:
    """Largest deviation from the fp64 oracle (ref_rows) of N_MODEL fp32-model runs
    on instances `rows` of `problem`, per quantity."""
    from oracle import Oracle
    if P is None:
        P, _, _ = bpoly_basis(oracle.params.q, oracle.params.T, oracle.params.degree)
    rows = np.asarray(rows)
    init = np.asarray(problem["init"], np.float64)[rows]
    lam = None if lambda_in is None else np.asarray(lambda_in, np.float64)[rows]
    seeds = range(MODEL_SEED0, MODEL_SEED0 + N_MODEL) if seeds is None else seeds
    spread = {}
    for s in seeds:
        om = Oracle(dataclasses.replace(oracle.params, fp32_model=1, noise_seed=int(s)), oracle.n)
        m = om.solve(problem["bnd"], problem["obs_xy"], problem["obs_ab"], init, iters, lambda_in=lam)
        for k, v in deviations(P, m, ref_rows).items():
            spread[k] = np.maximum(spread.get(k, 0.0), v)
    return spread


def _take(d: dict, rows) -> dict:
    out = {}
    for k, v in d.items():
        if isinstance(v, np.ndarray) and v.ndim >= 1 and k not in ("best",):
            out[k] = v[rows]
    return out


def compare(cfg, gpu: dict, ref: dict, tau: float, label: str = "", check_best: bool = True,
            oracle=None, problem=None, iters=None, lambda_in=None, idx=None) -> dict:
    """Element-by-element bar; instances that miss it are re-examined with the fp32
    rounding model when `oracle` and `problem` are given (idx maps the rows of
    gpu / ref to instances of problem)."""
    P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    iters = cfg.K if iters is None else iters
    dev = deviations(P, gpu, ref)
    bar = bars(cfg, ref, iters)
    n = len(dev["traj"])
    fails = {k: dev[k] > bar[k] for k in dev if k in bar}
    bad = np.flatnonzero(np.any(np.stack(list(fails.values())), axis=0))
    Jr = np.asarray(ref["cost"], np.float64)
    stats = dict(label=label, n=n, **{f"max_d{k}": float(v.max()) for k, v in dev.items()},
                 worst_inst=int(dev["traj"].argmax()),
                 max_rel_dJ=float(np.max(dev["cost"] / (np.abs(Jr) + 1e-12))), fp32_model_accepted=[])
    if bad.size and oracle is not None and problem is not None:
        rows = bad if idx is None else np.asarray(idx)[bad]
        sp = fp32_spread(oracle, problem, rows, iters, _take(ref, bad), lambda_in=lambda_in, P=P)
        keep = []
        for i, b in enumerate(bad):
            failing = [k for k in fails if fails[k][b]]
            ratios = {k: float(dev[k][b] / max(sp[k][i], 1e-300)) for k in failing}
            if all(r <= KAPPA for r in ratios.values()):
                stats["fp32_model_accepted"].append(
                    dict(inst=int(b), **{f"d{k}": float(dev[k][b]) for k in failing},
                         **{f"spread_{k}": float(sp[k][i]) for k in failing},
                         max_ratio=max(ratios.values())))
            else:
                keep.append((int(b), {k: (float(dev[k][b]), float(bar[k][b]), float(sp[k][i])) for k in failing}))
        bad = np.array([b for b, _ in keep], dtype=int)
        stats["rejected"] = keep[:10]
    for a in stats["fp32_model_accepted"]:
        print(f"{label}: instance {a['inst']} accepted by the fp32 rounding model: {a}")
    msg = f"{label}: {stats}; failing instances {bad.tolist()[:10]}"
    assert bad.size == 0, msg
    if check_best and "best_index" in ref:
        gb = int(np.asarray(gpu["best"])[0])
        rb = ref["best_index"]
        stats["best"] = (gb, rb)
        if gb != rb:
            r1 = np.asarray(ref["residual"], np.float64)[:, 0]
            feas, v = key_value(r1, Jr, tau)
            near_tau = bool(np.any(np.abs(r1 - tau) <= 1e-3 * tau))
            order = np.lexsort((np.arange(len(v)), v, ~feas))
            close = (len(v) > 1 and feas[order[0]] == feas[order[1]]
                     and abs(float(v[order[1]]) - float(v[order[0]])) <= 1e-3 * abs(float(v[order[0]])))
            assert near_tau or close, f"{label}: best index gpu {gb} != oracle {rb} on an unambiguous scene"
            assert feas[gb] == feas[rb] and abs(float(v[gb]) - float(v[rb])) <= 1e-4 * abs(float(v[rb])), \
                f"{label}: ambiguous scene, but the GPU's pick {gb} is not within 1e-4 of the oracle's best {rb}"
    return stats
