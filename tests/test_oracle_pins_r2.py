"""Pins of the oracle's cost J, its multiplier steps and its QP steps at
non-default weights, each against something other than the oracle itself.

* cost J = sum_t (xdd^2 + ydd^2 + psidd^2) (Eq. 1a; reading G17):
  recomputed from the oracle's returned coefficients with scipy BPoly second
  derivatives, on instances whose heading has real curvature (so a dropped
  psidd^2 term, or a Pd / Pdd swap, fails);
* lambda_psi step (Eq. 23b; reading G4): Delta lambda_psi equals
  -rho_psi times the central finite-difference gradient of
  0.5 ||P xi2 - theta||^2 with P from BPoly, at rho = 0.5, rho_psi = 2 (so a
  rho / rho_psi mix-up fails);
* lambda step (Eq. 23a; reading G3) at rho = 0.5: Delta lambda equals
  -rho times the finite-difference gradient of 0.5 ||F xi1 - g||^2 with the
  rows of F rebuilt pointwise from BPoly trajectories (Eq. 10-11);
* xi1 / xi2 steps (Eq. 3-4, 17, 19) at rho != rho_psi, w_copy > 0 (G10) and
  boundary masks != 0x3F (G11) against numpy.linalg.solve of KKT systems
  assembled from the BPoly basis.
"""
import numpy as np
import pytest

from oracle import Oracle
from synth import CONFIGS, make_problem
from tests.helpers import bpoly_basis, eval_bpoly, oracle_params

RHO, RHO_PSI = 0.5, 2.0


def _bnd_curved():
    """Boundary with a turning heading and a lateral offset (psi has curvature)."""
    b = make_problem(CONFIGS["C3"].with_(n=0), 0, B=1)["bnd"].copy()
    b[1] = [0.0, 0.2, 0.0, 1.5, -0.1, 0.0]
    b[2] = [0.3, 0.02, 0.0, -0.4, 0.0, 0.001]
    return b


def _J_bpoly(coeffs, T, q):
    t = np.linspace(0.0, T, q)
    J = np.zeros(coeffs.shape[0])
    terms = np.zeros((coeffs.shape[0], 3))
    for l in range(coeffs.shape[0]):
        for i, blk in enumerate((0, 2, 4)):
            terms[l, i] = np.sum(eval_bpoly(coeffs[l, blk], T, t, 2) ** 2)
        J[l] = terms[l].sum()
    return J, terms


@pytest.mark.parametrize("K", [0, 3, 12])
def test_cost_J_is_sum_of_squared_second_derivatives(K):
    cfg = CONFIGS["C3"].with_(n=4, q=60)
    pr = make_problem(cfg, 3, B=6)
    bnd = _bnd_curved()
    init = pr["init"].astype(np.float64)
    rng = np.random.default_rng(17)
    init[:, 2] = np.linspace(bnd[2, 0], bnd[2, 3], 11) + 0.4 * rng.standard_normal((6, 11))  # curved c_psi
    o = Oracle(oracle_params(cfg, rho=RHO, rho_psi=RHO_PSI), cfg.n)
    out = o.solve(bnd, pr["obs_xy"], pr["obs_ab"], init, K)
    J, terms = _J_bpoly(out["coeffs"], cfg.T, cfg.q)
    assert np.allclose(out["cost"], J, rtol=1e-10, atol=0.0)
    # the heading term is a real part of J here: dropping it would fail the check above
    assert np.all(terms[:, 2] > 1e-6 * J)
    # Pd instead of Pdd would give a different number (sanity of the pin's sensitivity)
    t = np.linspace(0.0, cfg.T, cfg.q)
    Jd = sum(np.sum(eval_bpoly(out["coeffs"][0, b], cfg.T, t, 1) ** 2) for b in (0, 2, 4))
    assert abs(Jd - J[0]) > 1e-3 * J[0]


@pytest.fixture(scope="module")
def weighted_trace():
    cfg = CONFIGS["C3"].with_(n=5, q=40, rho=RHO, rho_psi=RHO_PSI)
    pr = make_problem(cfg, 2, B=3)
    bnd = _bnd_curved()
    o = Oracle(oracle_params(cfg), cfg.n)
    tr = o.trace_instance(bnd, pr["obs_xy"], pr["obs_ab"], pr["init"][1], 8)
    return cfg, pr, bnd, o, tr


def test_lampsi_step_is_fd_gradient(weighted_trace):
    """Eq. 23b with the gradient-consistent sign (G4) and rho_psi in the step (G5)."""
    cfg, pr, bnd, o, tr = weighted_trace
    P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    nonzero = 0
    for k in range(1, 9):
        xi2, theta = tr["xi2"][k], tr["theta"][k]
        f = lambda z: 0.5 * np.sum((P @ z - theta) ** 2)
        h = 1e-6
        grad = np.array([(f(xi2 + h * e) - f(xi2 - h * e)) / (2 * h) for e in np.eye(11)])
        dlam = tr["lam"][k][44:] - tr["lam"][k - 1][44:]
        assert np.allclose(dlam, -RHO_PSI * grad, rtol=1e-6, atol=1e-8 * max(1.0, np.abs(grad).max()))
        nonzero += np.abs(grad).max() > 1e-6
    assert nonzero >= 4   # the heading residual is active on this scene


def _penalty_bpoly(cfg, xi, g):
    """0.5 ||F xi - g||^2 with F's rows (Eq. 10-11) evaluated pointwise from BPoly."""
    q, m, n = cfg.q, cfg.m, cfg.n
    t = np.linspace(0.0, cfg.T, q)
    R = 2 * q + m * n * q + q
    tot = 0.0
    for ch in range(2):
        pos, cop = xi[ch * 22:ch * 22 + 11], xi[ch * 22 + 11:ch * 22 + 22]
        gg = g[ch * R:(ch + 1) * R]
        p, pd, pdd = (eval_bpoly(pos, cfg.T, t, nu) for nu in (0, 1, 2))
        cc = eval_bpoly(cop, cfg.T, t)
        tot += np.sum((pd - gg[:q]) ** 2) + np.sum((pdd - gg[q:2 * q]) ** 2)
        for j in range(n):
            for i in range(m):
                r0 = 2 * q + (j * m + i) * q
                tot += np.sum((p + cfg.offsets[i] * cc - gg[r0:r0 + q]) ** 2)
        tot += np.sum((cc - gg[2 * q + m * n * q:]) ** 2)
    return 0.5 * tot


def test_lambda_step_is_fd_gradient_rho_half(weighted_trace):
    cfg, pr, bnd, o, tr = weighted_trace
    for k in (2, 5, 8):
        xi, g = tr["xi1"][k], tr["g"][k]
        h = 1e-5
        grad = np.array([(_penalty_bpoly(cfg, xi + h * e, g) - _penalty_bpoly(cfg, xi - h * e, g)) / (2 * h)
                         for e in np.eye(44)])
        dlam = tr["lam"][k][:44] - tr["lam"][k - 1][:44]
        assert np.allclose(dlam, -RHO * grad, rtol=1e-5, atol=1e-7 * max(1.0, np.abs(grad).max()))


def _A_rows(P, Pd, Pdd, mask):
    rows = []
    for bit in range(6):
        if mask & (1 << bit):
            src = (P, Pd, Pdd)[bit % 3]
            rows.append(src[0] if bit < 3 else src[-1])
    return np.array(rows).reshape(-1, P.shape[1])


@pytest.mark.parametrize("rho,rho_psi,w_copy,mask", [(0.5, 2.0, 0.0, 0x3F), (1.0, 1.0, 0.1, 0x3F),
                                                      (0.5, 2.0, 0.1, 0x09), (1.0, 1.0, 0.0, 0x1B),
                                                      (2.0, 0.5, 0.0, 0x07)])
def test_qp_steps_at_nondefault_weights(rho, rho_psi, w_copy, mask):
    cfg = CONFIGS["C3"].with_(n=3, q=50)
    o = Oracle(oracle_params(cfg, rho=rho, rho_psi=rho_psi, w_copy=w_copy, boundary_mask=mask), cfg.n)
    rng = np.random.default_rng(mask + int(10 * rho))
    P, Pd, Pdd = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    A = _A_rows(P, Pd, Pdd, mask)
    nb = A.shape[0]
    bnd = _bnd_curved()
    sel = [bit for bit in range(6) if mask & (1 << bit)]
    F = o.F
    lam = rng.standard_normal(44)
    g = F @ rng.standard_normal(44) + 0.3 * rng.standard_normal(F.shape[0])
    xi = o.xi1_step(lam, g, bnd)
    Qs = Pdd.T @ Pdd
    Q = np.zeros((44, 44))
    for blk, w in ((0, 1.0), (1, w_copy), (2, 1.0), (3, w_copy)):
        Q[blk * 11:(blk + 1) * 11, blk * 11:(blk + 1) * 11] = w * Qs
    Af = np.zeros((2 * nb, 44))
    Af[:nb, :11] = A
    Af[nb:, 22:33] = A
    b = np.concatenate([bnd[0, sel], bnd[1, sel]])
    Kmat = np.block([[Q + rho * F.T @ F, Af.T], [Af, np.zeros((2 * nb, 2 * nb))]])
    ref = np.linalg.solve(Kmat, np.concatenate([lam + rho * F.T @ g, b]))[:44]
    assert np.max(np.abs(xi - ref)) < 1e-8 * max(1, np.abs(ref).max())
    assert np.max(np.abs(Af @ xi - b)) < 1e-9
    theta = 0.3 * rng.standard_normal(cfg.q)
    lampsi = rng.standard_normal(11)
    xi2 = o.xi2_step(lampsi, theta, bnd)
    H = Pdd.T @ Pdd + rho_psi * P.T @ P
    Kp = np.block([[H, A.T], [A, np.zeros((nb, nb))]])
    ref2 = np.linalg.solve(Kp, np.concatenate([lampsi + rho_psi * P.T @ theta, bnd[2, sel]]))[:11]
    assert np.max(np.abs(xi2 - ref2)) < 1e-8 * max(1, np.abs(ref2).max())


@pytest.mark.parametrize("rho,rho_psi", [(0.5, 2.0), (2.0, 0.5)])
def test_obstacle_free_fixed_point_any_weights(rho, rho_psi):
    """The closed-form minimum-acceleration QP is a fixed point for any penalty weights."""
    cfg = CONFIGS["C1"].with_(n=0, v_max=100.0, a_max=100.0)
    P, Pd, Pdd = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    A = np.vstack([P[0], Pd[0], Pdd[0], P[-1], Pd[-1], Pdd[-1]])
    bnd = np.array([[0.0, 1.2, 0.05, 28.0, 0.8, -0.02], [0.0, 0.3, 0.0, 2.0, -0.2, 0.01],
                    [0.2, 0.0, 0.0, 0.2, 0.0, 0.0]])
    K = np.block([[Pdd.T @ Pdd, A.T], [A, np.zeros((6, 6))]])
    cx, cy = (np.linalg.solve(K, np.concatenate([np.zeros(11), bnd[ch]]))[:11] for ch in (0, 1))
    o = Oracle(oracle_params(cfg, rho=rho, rho_psi=rho_psi), 0)
    tr = o.trace_instance(bnd, None, None, np.stack([cx, cy, np.full(11, 0.2)]), 6)
    for k in range(1, 7):
        assert np.max(np.abs(tr["xi1"][k][:11] - cx)) < 3e-8
        assert np.max(np.abs(tr["xi1"][k][22:33] - cy)) < 3e-8
        assert np.max(np.abs(tr["lam"][k])) < 1e-9
