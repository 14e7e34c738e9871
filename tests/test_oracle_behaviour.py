"""Whole-iteration pins of the oracle (no worked iterate is printed in the paper).

* obstacle-free exact fixed point = the closed-form minimum-acceleration QP
  (numpy KKT on the BPoly basis), plus monotone approach from a perturbed init;
* translation and mirror equivariance, batch independence and permutation;
* single circle r = 0 decouples the heading sub-problem;
* worked scene: monotone r1 decay to the fp64 floor (BASELINE north_star);
* G4 decision: the printed lambda_psi sign (Eq. 23b) diverges, the
  gradient-consistent sign does not.
"""
import numpy as np
import pytest

from oracle import Oracle
from synth import CONFIGS, make_init, make_problem
from tests.helpers import bpoly_basis, eval_bpoly, oracle_params


def _min_acc_qp(cfg, bnd):
    P, Pd, Pdd = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    A = np.vstack([P[0], Pd[0], Pdd[0], P[-1], Pd[-1], Pdd[-1]])
    H = Pdd.T @ Pdd
    K = np.block([[H, A.T], [A, np.zeros((6, 6))]])
    return [np.linalg.solve(K, np.concatenate([np.zeros(11), bnd[ch]]))[:11] for ch in (0, 1)]


BND_FREE = np.array([[0.0, 1.2, 0.05, 28.0, 0.8, -0.02],
                     [0.0, 0.3, 0.0, 2.0, -0.2, 0.01],
                     [0.2, 0.0, 0.0, 0.2, 0.0, 0.0]])


def test_obstacle_free_fixed_point():
    cfg = CONFIGS["C1"].with_(n=0, v_max=100.0, a_max=100.0)
    cx, cy = _min_acc_qp(cfg, BND_FREE)
    psi0 = BND_FREE[2, 0]
    init = np.stack([cx, cy, np.full(11, psi0)])
    o = Oracle(oracle_params(cfg), 0)
    tr = o.trace_instance(BND_FREE, None, None, init, 8)
    expect = np.concatenate([cx, np.full(11, np.cos(psi0)), cy, np.full(11, np.sin(psi0))])
    for k in range(1, 9):
        assert np.max(np.abs(tr["xi1"][k] - expect)) < 1e-9 * 30
        assert np.max(np.abs(tr["xi2"][k] - psi0)) < 1e-9
        assert np.max(np.abs(tr["lam"][k])) < 1e-9
        assert tr["r1"][k] < 1e-9


def test_obstacle_free_approach_is_monotone():
    cfg = CONFIGS["C1"].with_(n=0, v_max=100.0, a_max=100.0)
    cx, cy = _min_acc_qp(cfg, BND_FREE)
    rng = np.random.default_rng(9)
    init = np.stack([cx, cy, np.full(11, BND_FREE[2, 0])])
    init[0, 3:8] += rng.normal(0, 1.0, 5)
    init[1, 3:8] += rng.normal(0, 3.0, 5)
    o = Oracle(oracle_params(cfg), 0)
    K = 60
    tr = o.trace_instance(BND_FREE, None, None, init, K)
    F = o.F
    star = np.concatenate([cx, np.zeros(11), cy, np.zeros(11)])
    mask = np.zeros(44)
    mask[:11] = 1
    mask[22:33] = 1
    err = [np.linalg.norm(F @ ((tr["xi1"][k] - star) * mask)) for k in range(1, K + 1)]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(err, err[1:]))   # proximal-point metric
    t = np.linspace(0, cfg.T, cfg.q)
    d0 = np.max(np.abs(eval_bpoly(tr["xi1"][1][22:33] - cy, cfg.T, t)))
    dK = np.max(np.abs(eval_bpoly(tr["xi1"][K][22:33] - cy, cfg.T, t)))
    assert dK < 0.5 * d0


@pytest.fixture(scope="module")
def c3_scene():
    cfg = CONFIGS["C3"].with_(n=8, q=60, K=25)
    pr = make_problem(cfg, 4, B=5)
    o = Oracle(oracle_params(cfg), cfg.n)
    ref = o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K)
    return cfg, pr, o, ref


def test_translation_equivariance(c3_scene):
    cfg, pr, o, ref = c3_scene
    dx, dy = 3.25, -1.5
    bnd = pr["bnd"].copy()
    bnd[0, [0, 3]] += dx
    bnd[1, [0, 3]] += dy
    obs = pr["obs_xy"].astype(np.float64)
    obs[:, 0] += dx
    obs[:, 1] += dy
    init = pr["init"].astype(np.float64)
    init[:, 0] += dx          # partition of unity: adding a constant to all control points
    init[:, 1] += dy
    out = o.solve(bnd, obs, pr["obs_ab"], init, cfg.K)
    shift = np.zeros((5, 11))
    shift[0] = dx
    shift[2] = dy
    assert np.allclose(out["coeffs"], ref["coeffs"] + shift, atol=2e-8)
    assert np.allclose(out["cost"], ref["cost"], rtol=1e-6, atol=1e-10)
    assert np.allclose(out["residual"], ref["residual"], rtol=1e-6, atol=1e-10)


def test_mirror_equivariance(c3_scene):
    cfg, pr, o, ref = c3_scene
    bnd = pr["bnd"].copy()
    bnd[1] *= -1
    bnd[2] *= -1
    obs = pr["obs_xy"].astype(np.float64)
    obs[:, 1] *= -1
    init = pr["init"].astype(np.float64)
    init[:, 1:] *= -1
    out = o.solve(bnd, obs, pr["obs_ab"], init, cfg.K)
    sgn = np.array([1, 1, -1, -1, -1])[:, None]
    assert np.allclose(out["coeffs"], ref["coeffs"] * sgn, atol=1e-8)
    assert np.allclose(out["lambda_out"], ref["lambda_out"] * sgn, atol=1e-8)
    assert np.allclose(out["cost"], ref["cost"], rtol=1e-8)


def test_batch_independence_and_permutation(c3_scene):
    cfg, pr, o, ref = c3_scene
    perm = np.array([3, 0, 4, 1, 2])
    out = o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"][perm], cfg.K)
    assert np.array_equal(out["coeffs"], ref["coeffs"][perm])
    assert np.array_equal(out["residual"], ref["residual"][perm])
    one = o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"][2:3], cfg.K)
    assert np.array_equal(one["coeffs"][0], ref["coeffs"][2])


def test_best_index_rule(c3_scene):
    cfg, pr, o, ref = c3_scene
    r1, J = ref["residual"][:, 0], ref["cost"]
    feas = r1 <= cfg.res_tol
    if feas.any():
        cand = np.where(feas)[0]
        expect = cand[np.argmin(J[cand].astype(np.float32))]
    else:
        expect = int(np.argmin(r1.astype(np.float32)))
    assert ref["best_index"] == expect
    assert (ref["best_key"] >> 62) == (0 if feas.any() else 1)


def test_single_circle_decouples_heading():
    """m = 1, r = 0: collision rows do not involve c, s, so (c_x, c_y) are
    independent of the heading sub-problem's weight rho_psi."""
    cfg = CONFIGS["C1"].with_(m=1, n=3)
    pr = make_problem(cfg, 1, B=3)
    outs = []
    for rp in (0.5, 3.0):
        o = Oracle(oracle_params(cfg, r=[0.0], rho_psi=rp), cfg.n)
        outs.append(o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], 20))
    a, b = outs
    assert np.allclose(a["coeffs"][:, [0, 2]], b["coeffs"][:, [0, 2]], atol=1e-12, rtol=0)


def _worked_scene(m, yob=0.3):
    cfg = CONFIGS["C1"].with_(n=1, B=16, K=50, m=m)
    obs = np.zeros((1, 2, cfg.q), np.float32)
    obs[0, 0] = 15.0
    obs[0, 1] = yob
    ab = np.full((1, 2), 0.6, np.float32)
    init = make_init(cfg, 7, B=16)
    return cfg, obs, ab, init


def test_worked_scene_monotone_residual_decay():
    """One static circular obstacle near the straight line, B = 16, q = 50, K = 50,
    single circle (r = 0): r1 is non-increasing from k >= 1 until it reaches the fp64
    floor (1e-9), and every instance ends below 1e-8."""
    cfg, obs, ab, init = _worked_scene(1)
    o = Oracle(oracle_params(cfg, r=[0.0]), 1)
    out = o.solve(np.asarray(make_problem(cfg, 0, B=1)["bnd"]), obs, ab, init, cfg.K, trace=True)
    tr = out["res_trace"]
    n_active = 0
    for l in range(16):
        r = tr[l]
        if r[0] > 1e-6:
            n_active += 1
        above = r > 1e-9
        for k in range(1, cfg.K):
            if above[k]:
                assert r[k] <= r[k - 1] * (1 + 1e-12), (l, k, r[k - 1], r[k])
        assert r[-1] < 1e-8
    assert n_active >= 2


def test_lampsi_sign_reading_G4():
    """The printed Eq. 23b sign makes the heading residual blow up on the worked scene with
    two circles; the gradient-consistent sign keeps it small."""
    cfg, obs, ab, init = _worked_scene(2)
    bnd = make_problem(cfg, 0, B=1)["bnd"]
    res = {}
    for sign in (0, 1):
        o = Oracle(oracle_params(cfg, lampsi_printed_sign=sign), 1)
        tr = o.trace_instance(bnd, obs, ab, init[0], 40)
        res[sign] = tr["rpsi"]
    assert res[0][-1] < 1e-2 and np.all(np.isfinite(res[0]))
    assert res[1][-1] > 1e3 * max(res[0][-1], 1e-6)
