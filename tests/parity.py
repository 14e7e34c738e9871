"""GPU <-> oracle comparison used by the -m gpu tests and smoke().

Tolerances (BASELINE.json north_star):
  * trajectory: max over t and the x, y channels of |P (c_gpu - c_oracle)| <= 1e-3 m,
    with P the fp64 basis (scipy BPoly, independent of both sides);
  * cost J: |dJ| <= 1e-4 |J| + 1e-8 q;
  * residuals r1, r_psi: |dr| <= 1e-4 |r| + RES_FLOOR, RES_FLOOR = 2e-5: the GPU
    evaluates trajectories in fp32, so each residual row carries ~1e-7 absolute
    rounding and ||.||_2 over ~1e4 rows an absolute floor of ~1e-5;
  * best index identical, unless the scene is ambiguous (a residual within 1e-3
    relative of tau, or the oracle's best and runner-up keys within 1e-3
    relative): then the GPU's pick must be within 1e-4 of the oracle's best value.
"""
from __future__ import annotations

import numpy as np

from tests.helpers import bpoly_basis

TRAJ_TOL = 1e-3
COST_RTOL = 1e-4
RES_RTOL = 1e-4
RES_FLOOR = 2e-5


def key_value(r1, J, tau):
    feas = r1 <= tau
    v = np.where(feas, J, r1).astype(np.float32)
    return feas, v


def compare(cfg, gpu: dict, ref: dict, tau: float, label: str = "", check_best: bool = True,
            traj_tol: float = TRAJ_TOL) -> dict:
    P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    cg = np.asarray(gpu["coeffs"], dtype=np.float64)
    cr = np.asarray(ref["coeffs"], dtype=np.float64)
    dtraj = np.zeros(cg.shape[0])
    for blk in (0, 2):
        dtraj = np.maximum(dtraj, np.max(np.abs((cg[:, blk] - cr[:, blk]) @ P.T), axis=1))
    dpsi = np.max(np.abs((cg[:, 4] - cr[:, 4]) @ P.T), axis=1)
    Jg, Jr = np.asarray(gpu["cost"], np.float64), np.asarray(ref["cost"], np.float64)
    rg, rr = np.asarray(gpu["residual"], np.float64), np.asarray(ref["residual"], np.float64)
    dJ = np.abs(Jg - Jr)
    dr = np.abs(rg - rr)
    stats = dict(label=label, max_dtraj=float(dtraj.max()), max_dpsi=float(dpsi.max()),
                 worst_inst=int(dtraj.argmax()),
                 max_rel_dJ=float(np.max(dJ / (np.abs(Jr) + 1e-12))),
                 max_dr=float(dr.max()))
    bad_t = np.where(dtraj > traj_tol)[0]
    bad_J = np.where(dJ > COST_RTOL * np.abs(Jr) + 1e-8 * cfg.q)[0]
    bad_r = np.where(np.any(dr > RES_RTOL * np.abs(rr) + RES_FLOOR, axis=1))[0]
    msg = (f"{label}: {stats}; traj fails {bad_t.tolist()[:10]}, cost fails {bad_J.tolist()[:10]}, "
           f"residual fails {bad_r.tolist()[:10]}")
    assert bad_t.size == 0 and bad_J.size == 0 and bad_r.size == 0, msg
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
            assert ambiguous, f"{label}: best index gpu {gb} != oracle {rb} on an unambiguous scene"
            assert abs(float(v[gb]) - float(v[rb])) <= 1e-4 * abs(float(v[rb])) + 1e-12
    return stats
