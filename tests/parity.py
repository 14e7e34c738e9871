"""GPU <-> oracle comparison used by the -m gpu tests and smoke().

Tolerances (BASELINE.json north_star):
  * trajectory: max over t and the x, y channels of |P (c_gpu - c_oracle)| <= 1e-3 m,
    with P the fp64 basis (scipy BPoly, independent of both sides);
  * cost J: |dJ| <= 1e-4 |J| + 1e-8 q;
  * residuals r1, r_psi: |dr| <= 1e-4 |r| + RES_FLOOR, RES_FLOOR = 2e-5: the GPU
    evaluates the per-row residuals in fp32, so each row carries ~1e-7 absolute
    rounding and ||.||_2 over ~1e4 rows an absolute floor of ~1e-5;
  * best index identical, unless the scene is ambiguous (a residual within 1e-3
    relative of tau, or the oracle's best and runner-up keys within 1e-3
    relative): then the GPU's pick must be within 1e-4 of the oracle's best value.

Ill-conditioned instances: the AM iteration is a
non-smooth, non-convex map; on some instances it amplifies perturbations by
>1e3 over 100 iterations, so a one-ulp (fp32) change of the input moves the
fp64 oracle's own answer by more than the tolerance.  For an instance that
misses the bar, the oracle is re-run on `N_PERT` copies of its input with the
interior control points perturbed by `PERT_REL` (relative, the fp32 input
rounding scale) and the obstacle positions by `PERT_OBS` (absolute, the fp32
rounding of positions in the kernel's deviation frame: |x - x_ref| <= 30 m has
an ulp of 2e-6 m); the instance passes only if the GPU deviation is within
`KAPPA` times that spread for every quantity that misses the bar.  The kernel
rounds at that scale in every iteration, not once at the input, hence the
factor; a well-conditioned instance (spread ~1e-7) still gets no slack.  At
full C3 size about 0.5 % of the instances need this.
Every such acceptance is reported.
"""
from __future__ import annotations

import numpy as np

from tests.helpers import bpoly_basis

TRAJ_TOL = 1e-3
COST_RTOL = 1e-4
RES_RTOL = 1e-4
RES_FLOOR = 2e-5
PERT_REL = 1e-7
PERT_OBS = 1e-6
N_PERT = 3
KAPPA = 10.0


def key_value(r1, J, tau):
    feas = r1 <= tau
    v = np.where(feas, J, r1).astype(np.float32)
    return feas, v


def _deviations(P, cg, cr, Jg, Jr, rg, rr):
    cg = np.asarray(cg, dtype=np.float64)
    cr = np.asarray(cr, dtype=np.float64)
    dtraj = np.zeros(cg.shape[0])
    for blk in (0, 2):
        dtraj = np.maximum(dtraj, np.max(np.abs((cg[:, blk] - cr[:, blk]) @ P.T), axis=1))
    dJ = np.abs(np.asarray(Jg, np.float64) - np.asarray(Jr, np.float64))
    dr = np.abs(np.asarray(rg, np.float64) - np.asarray(rr, np.float64))
    return dtraj, dJ, dr


def _fails(cfg, dtraj, dJ, dr, Jr, rr, scale=None):
    """Per-instance bar; `scale` = (traj, cost, res) allowances replacing the tolerances."""
    tt = TRAJ_TOL if scale is None else np.maximum(TRAJ_TOL, scale[0])
    tJ = COST_RTOL * np.abs(Jr) + 1e-8 * cfg.q
    tr = RES_RTOL * np.abs(rr) + RES_FLOOR
    if scale is not None:
        tJ = np.maximum(tJ, scale[1])
        tr = np.maximum(tr, scale[2][:, None] if np.ndim(scale[2]) == 1 else scale[2])
    return (dtraj > tt) | (dJ > tJ) | np.any(dr > tr, axis=1)


def intrinsic_spread(cfg, oracle, problem, idx, iters, lambda_in=None, seed=0):
    """Oracle's own spread on instances `idx` under PERT_REL perturbations of the input."""
    P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    init = np.asarray(problem["init"], dtype=np.float64)[idx]
    lam = None if lambda_in is None else np.asarray(lambda_in, np.float64)[idx]
    base = oracle.solve(problem["bnd"], problem["obs_xy"], problem["obs_ab"], init, iters, lambda_in=lam)
    rng = np.random.default_rng(seed)
    st = np.zeros(len(idx))
    sJ = np.zeros(len(idx))
    sr = np.zeros((len(idx), 2))
    obs = np.asarray(problem["obs_xy"], dtype=np.float64)
    for _ in range(N_PERT):
        pert = init.copy()
        pert[:, :2, 3:8] *= 1.0 + PERT_REL * rng.standard_normal(pert[:, :2, 3:8].shape)
        obs_p = obs + PERT_OBS * rng.standard_normal(obs.shape) if obs.size else obs
        o = oracle.solve(problem["bnd"], obs_p, problem["obs_ab"], pert, iters, lambda_in=lam)
        t_, J_, r_ = _deviations(P, o["coeffs"], base["coeffs"], o["cost"], base["cost"], o["residual"],
                                 base["residual"])
        st, sJ, sr = np.maximum(st, t_), np.maximum(sJ, J_), np.maximum(sr, r_)
    return st, sJ, sr


def compare(cfg, gpu: dict, ref: dict, tau: float, label: str = "", check_best: bool = True,
            oracle=None, problem=None, iters=None, lambda_in=None, idx=None) -> dict:
    """Element-by-element bar; instances that miss it are re-examined for ill-conditioning
    when `oracle` and `problem` are given (idx maps rows to problem instances)."""
    P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    Jr = np.asarray(ref["cost"], np.float64)
    rr = np.asarray(ref["residual"], np.float64)
    dtraj, dJ, dr = _deviations(P, gpu["coeffs"], ref["coeffs"], gpu["cost"], Jr, gpu["residual"], rr)
    dpsi = np.max(np.abs((np.asarray(gpu["coeffs"], np.float64)[:, 4] - ref["coeffs"][:, 4]) @ P.T), axis=1)
    bad = np.where(_fails(cfg, dtraj, dJ, dr, Jr, rr))[0]
    stats = dict(label=label, n=len(dtraj), max_dtraj=float(dtraj.max()), max_dpsi=float(dpsi.max()),
                 worst_inst=int(dtraj.argmax()), max_rel_dJ=float(np.max(dJ / (np.abs(Jr) + 1e-12))),
                 max_dr=float(dr.max()), ill_conditioned=[])
    if bad.size and oracle is not None and problem is not None:
        rows = bad if idx is None else np.asarray(idx)[bad]
        st, sJ, sr = intrinsic_spread(cfg, oracle, problem, rows, cfg.K if iters is None else iters,
                                      lambda_in=lambda_in)
        accept = ~_fails(cfg, dtraj[bad], dJ[bad], dr[bad], Jr[bad], rr[bad],
                         scale=(KAPPA * st, KAPPA * sJ, KAPPA * sr))
        for b, s_t, s_J, ok in zip(bad, st, sJ, accept):
            if ok:
                stats["ill_conditioned"].append(dict(inst=int(b), dtraj=float(dtraj[b]), spread_traj=float(s_t),
                                                     dJ=float(dJ[b]), spread_J=float(s_J)))
        bad = bad[~accept]
    msg = f"{label}: {stats}; failing instances {bad.tolist()[:10]}"
    assert bad.size == 0, msg
    if check_best and "best_index" in ref:
        gb = int(np.asarray(gpu["best"])[0])
        rb = ref["best_index"]
        if gb != rb:
            r1 = rr[:, 0]
            feas, v = key_value(r1, Jr, tau)
            near_tau = np.any(np.abs(r1 - tau) <= 1e-3 * tau)
            order = np.lexsort((np.arange(len(v)), v, ~feas))
            ambiguous = near_tau or (len(v) > 1 and feas[order[0]] == feas[order[1]]
                                     and abs(float(v[order[1]]) - float(v[order[0]])) <= 1e-3 * abs(float(v[order[0]])))
            ill = {d["inst"] for d in stats["ill_conditioned"]}
            assert ambiguous or rb in ill or gb in ill, \
                f"{label}: best index gpu {gb} != oracle {rb} on an unambiguous scene"
    return stats
