"""Shared test helpers: independent references (scipy BPoly), parameter builders.

Nothing here re-implements the method: the basis comes from scipy's BPoly
(a library routine independent of oracle.c and of the CUDA setup code).
"""
from __future__ import annotations

import numpy as np
from scipy.interpolate import BPoly

from synth import Config


def bpoly_basis(q: int, T: float, degree: int):
    """P, Pd, Pdd [q][nv] from scipy.interpolate.BPoly (Bernstein on [0, T])."""
    nv = degree + 1
    t = np.linspace(0.0, T, q)
    P = np.zeros((q, nv))
    Pd = np.zeros((q, nv))
    Pdd = np.zeros((q, nv))
    for k in range(nv):
        c = np.zeros((nv, 1))
        c[k, 0] = 1.0
        bp = BPoly(c, [0.0, T])
        P[:, k] = bp(t)
        Pd[:, k] = bp.derivative(1)(t)
        Pdd[:, k] = bp.derivative(2)(t)
    return P, Pd, Pdd


def eval_bpoly(coef: np.ndarray, T: float, t: np.ndarray, nu: int = 0) -> np.ndarray:
    bp = BPoly(np.asarray(coef, dtype=np.float64).reshape(-1, 1), [0.0, T])
    return bp.derivative(nu)(t) if nu else bp(t)


def oracle_params(cfg: Config, **kw):
    from oracle import OracleParams
    args = dict(q=cfg.q, T=cfg.T, degree=cfg.degree, r=cfg.offsets, v_max=cfg.v_max,
                a_max=cfg.a_max, rho=cfg.rho, rho_psi=cfg.rho_psi, res_tol=cfg.res_tol)
    args.update(kw)
    return OracleParams(**args)


def boundary_values(coef_x, coef_y, coef_psi, T):
    """(p0, v0, a0, pT, vT, aT) per channel from the coefficients (BPoly)."""
    out = []
    for c in (coef_x, coef_y, coef_psi):
        vals = []
        for tt in (0.0, T):
            for nu in (0, 1, 2):
                vals.append(float(eval_bpoly(c, T, np.array([tt]), nu)[0]))
        out.append([vals[0], vals[1], vals[2], vals[3], vals[4], vals[5]])
    return np.array(out)
