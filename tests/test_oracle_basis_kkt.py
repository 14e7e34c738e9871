"""Pins of the oracle's problem construction against independent references.

* basis (Eq. 8): scipy BPoly (library), partition of unity,
  endpoint interpolation, central differences;
* F (Eq. 10-11): shape and row semantics checked
  against trajectories evaluated with BPoly;
* xi1 / xi2 steps (Eq. 3-4, 17, 19): numpy.linalg.solve of the KKT system,
  boundary equalities, stationarity and optimality against random feasible
  perturbations, generic sign example (G1).
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import Oracle
from synth import CONFIGS, make_problem
from tests.helpers import bpoly_basis, eval_bpoly, oracle_params

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("q,T,deg", [(50, 30.0, 10), (100, 30.0, 10), (12, 2.5, 5), (7, 1.0, 2)])
def test_basis_matches_bpoly(q, T, deg):
    P, Pd, Pdd = oracle.basis(q, T, deg)
    Pr, Pdr, Pddr = bpoly_basis(q, T, deg)
    assert np.max(np.abs(P - Pr)) < 1e-12
    assert np.max(np.abs(Pd - Pdr)) < 1e-12 * max(1.0, np.abs(Pdr).max())
    assert np.max(np.abs(Pdd - Pddr)) < 1e-12 * max(1.0, np.abs(Pddr).max())


def test_basis_identities():
    q, T, deg = 100, 30.0, 10
    P, Pd, Pdd = oracle.basis(q, T, deg)
    assert np.allclose(P.sum(1), 1.0, atol=1e-13)          # partition of unity
    assert np.allclose(Pd.sum(1), 0.0, atol=1e-13)
    assert np.allclose(Pdd.sum(1), 0.0, atol=1e-13)
    assert np.all(P >= 0.0)
    e0 = np.zeros(deg + 1); e0[0] = 1
    en = np.zeros(deg + 1); en[-1] = 1
    assert np.allclose(P[0], e0, atol=0) and np.allclose(P[-1], en, atol=0)
    dt = T / (q - 1)                                         # S:65 central differences, O(dt^2)
    fd = (P[2:] - P[:-2]) / (2 * dt)
    assert np.max(np.abs(fd - Pd[1:-1])) < 0.1 * dt ** 2
    fd2 = (Pd[2:] - Pd[:-2]) / (2 * dt)
    assert np.max(np.abs(fd2 - Pdd[1:-1])) < 0.1 * dt ** 2


@pytest.mark.parametrize("q,T,deg", [(5, 1.0, 10), (20, 1.0, 1), (20, 0.0, 10)])
def test_basis_invalid(q, T, deg):
    with pytest.raises(ValueError):
        oracle.basis(q, T, deg)


def test_F_shape_and_rows():
    g = GOLD["F_shape"][0]
    cfg = CONFIGS["C1"].with_(m=g["m"], n=g["n"], q=g["q"])
    o = Oracle(oracle_params(cfg), g["n"])
    F = o.F
    assert F.shape == (g["rows"], g["cols"])
    # collision rows of F xi equal x + r_i c pointwise; other blocks per Eq. 10
    rng = np.random.default_rng(3)
    xi = rng.standard_normal(44)
    t = np.linspace(0, cfg.T, cfg.q)
    cx, cc, cy, cs = xi[:11], xi[11:22], xi[22:33], xi[33:44]
    x, c = eval_bpoly(cx, cfg.T, t), eval_bpoly(cc, cfg.T, t)
    y, s = eval_bpoly(cy, cfg.T, t), eval_bpoly(cs, cfg.T, t)
    Fx = F @ xi
    q, m, n, R = cfg.q, cfg.m, cfg.n, F.shape[0] // 2
    for ch, (pos, cop) in enumerate([(cx, cc), (cy, cs)]):
        blk = Fx[ch * R:(ch + 1) * R]
        p_t, c_t = (x, c) if ch == 0 else (y, s)
        assert np.allclose(blk[:q], eval_bpoly(pos, cfg.T, t, 1), atol=1e-10)
        assert np.allclose(blk[q:2 * q], eval_bpoly(pos, cfg.T, t, 2), atol=1e-10)
        for j in range(n):
            for i in range(m):
                r0 = 2 * q + (j * m + i) * q
                assert np.allclose(blk[r0:r0 + q], p_t + cfg.offsets[i] * c_t, atol=1e-10)
        assert np.allclose(blk[2 * q + m * n * q:], c_t, atol=1e-10)


def test_kkt_generic_sign_reading():
    """G1: the KKT right-hand side is (-q_bar, b)."""
    for ex in GOLD["kkt_generic"]:
        Q = np.array(ex["Q"])
        qb = np.array(ex["qbar"])
        A = np.array(ex["A"]).reshape(-1, Q.shape[0])
        K = np.block([[Q, A.T], [A, np.zeros((A.shape[0], A.shape[0]))]])
        sol = np.linalg.solve(K, np.concatenate([-qb, np.array(ex["b"])]))
        assert np.allclose(sol[:Q.shape[0]], ex["xi"], atol=1e-14), ex["cite"]


@pytest.fixture(scope="module")
def c3_small():
    cfg = CONFIGS["C3"].with_(n=6)
    o = Oracle(oracle_params(cfg), cfg.n)
    pr = make_problem(cfg, 0, B=4)
    return cfg, o, pr


def test_kkt_inverse(c3_small):
    cfg, o, _ = c3_small
    for K, Kinv in ((o.kkt1, o.kkt1_inv), (o.kktpsi, o.kktpsi_inv)):
        E = K @ Kinv - np.eye(K.shape[0])
        assert np.max(np.abs(E)) < 1e-7, np.max(np.abs(E))


def test_xi1_step_vs_numpy_solve_and_optimality(c3_small):
    cfg, o, pr = c3_small
    rng = np.random.default_rng(11)
    F, nv, nb = o.F, o.nv, o.nb
    lam = rng.standard_normal(4 * nv)
    g = F @ rng.standard_normal(4 * nv) + 0.3 * rng.standard_normal(F.shape[0])
    bnd = pr["bnd"]
    xi = o.xi1_step(lam, g, bnd)
    # independent: Q from BPoly, Q_bar = Q + rho F^T F, dense numpy solve of Eq. 3 (G1 sign)
    P, Pd, Pdd = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    Qs = Pdd.T @ Pdd
    Q = np.zeros((44, 44))
    Q[:11, :11] = Qs
    Q[22:33, 22:33] = Qs
    Qbar = Q + cfg.rho * F.T @ F
    A = np.vstack([P[0], Pd[0], Pdd[0], P[-1], Pd[-1], Pdd[-1]])
    Af = np.zeros((12, 44))
    Af[:6, :11] = A
    Af[6:, 22:33] = A
    b = np.concatenate([bnd[0], bnd[1]])
    Kmat = np.block([[Qbar, Af.T], [Af, np.zeros((12, 12))]])
    ref = np.linalg.solve(Kmat, np.concatenate([lam + cfg.rho * F.T @ g, b]))[:44]
    assert np.max(np.abs(xi - ref)) < 1e-8 * max(1, np.abs(ref).max())
    assert np.max(np.abs(Af @ xi - b)) < 1e-9                        # boundary
    # optimality of Eq. 13 against random feasible perturbations
    obj = lambda z: 0.5 * z @ Q @ z - lam @ z + 0.5 * cfg.rho * np.sum((F @ z - g) ** 2)
    _, _, Vt = np.linalg.svd(Af)
    N = Vt[12:].T                                                      # null space of A
    f0 = obj(xi)
    for _ in range(200):
        d = N @ rng.standard_normal(N.shape[1]) * 10 ** rng.uniform(-4, 0)
        assert obj(xi + d) >= f0 - 1e-9 * abs(f0)


def test_xi2_step_vs_numpy(c3_small):
    cfg, o, pr = c3_small
    rng = np.random.default_rng(5)
    theta = 0.3 * rng.standard_normal(cfg.q)
    lampsi = rng.standard_normal(11)
    bnd = pr["bnd"].copy()
    bnd[2] = [0.1, 0.0, 0.0, -0.2, 0.0, 0.0]
    xi2 = o.xi2_step(lampsi, theta, bnd)
    P, Pd, Pdd = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    A = np.vstack([P[0], Pd[0], Pdd[0], P[-1], Pd[-1], Pdd[-1]])
    H = Pdd.T @ Pdd + cfg.rho_psi * P.T @ P
    Kmat = np.block([[H, A.T], [A, np.zeros((6, 6))]])
    ref = np.linalg.solve(Kmat, np.concatenate([lampsi + cfg.rho_psi * P.T @ theta, bnd[2]]))[:11]
    assert np.max(np.abs(xi2 - ref)) < 1e-8 * max(1, np.abs(ref).max())
    assert np.max(np.abs(A @ xi2 - bnd[2])) < 1e-9


def test_constant_heading_target():
    """constant target theta = 0.3 with matching boundary -> psi(t) = 0.3."""
    cfg = CONFIGS["C1"]
    o = Oracle(oracle_params(cfg), 0)
    bnd = np.zeros((3, 6))
    bnd[2] = [0.3, 0, 0, 0.3, 0, 0]
    xi2 = o.xi2_step(np.zeros(11), np.full(cfg.q, 0.3), bnd)
    assert np.allclose(o.P @ xi2, 0.3, atol=1e-9)


def test_invalid_params():
    cfg = CONFIGS["C1"]
    for kw in (dict(q=5), dict(degree=1), dict(T=0.0), dict(rho=0.0), dict(v_max=-1.0),
               dict(boundary_mask=0x40)):
        with pytest.raises(ValueError):
            Oracle(oracle_params(cfg, **kw), 2)
    with pytest.raises(ValueError):   # rank-deficient boundary: 6 rows but q = nv... use degree 2
        Oracle(oracle_params(cfg, degree=2, q=3), 0)
