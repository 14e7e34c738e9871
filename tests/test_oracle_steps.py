"""Pins of the oracle's closed-form sub-steps and multiplier update.

* alpha / d projections (Eq. 21-22) against brute-force grids
   and the cited closed-form examples (golden file);
* lambda step (Eq. 23a with F^T, G3) against -rho x finite-difference
  gradient of 0.5 ||F xi - g||^2; zero residual -> unchanged;
* residual r1 = ||F xi1 - g|| against a pointwise recomputation of the
  Eq. 7c-7g violations from BPoly-evaluated trajectories.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import Oracle
from synth import CONFIGS, make_problem
from tests.helpers import eval_bpoly, oracle_params

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_golden_projections():
    for ex in GOLD["obstacle_projection"]:
        al, d = oracle.project_obstacle(ex["xt"], ex["yt"], ex["a"], ex["b"], ex["rule"])
        assert abs(al - ex["alpha"]) < 1e-12 and abs(d - ex["d"]) < 1e-9, ex["cite"]
        if "offset" in ex:
            off = (ex["a"] * d * np.cos(al), ex["b"] * d * np.sin(al))
            assert np.allclose(off, ex["offset"], atol=1e-9), ex["cite"]
    for ex in GOLD["bound_projection"]:
        al, d = oracle.project_bound(ex["vx"], ex["vy"], ex["bound"])
        assert abs(al - ex["alpha"]) < 1e-12 and abs(d - ex["d"]) < 1e-12, ex["cite"]


def _angle_diff(a, b):
    return abs((a - b + np.pi) % (2 * np.pi) - np.pi)


def test_alpha_step_equals_angle_grid_minimiser_circular():
    """for a = b and fixed d, atan2(yt, xt) minimises Eq. 20a over 1e4 angles."""
    rng = np.random.default_rng(0)
    grid = np.linspace(-np.pi, np.pi, 10000, endpoint=False)
    for _ in range(200):
        xt, yt = rng.uniform(-3, 3, 2)
        a = rng.uniform(0.2, 1.5)
        dprev = rng.uniform(1.0, 3.0)
        al, _ = oracle.project_obstacle(xt, yt, a, a, 0)
        cost = (xt - a * dprev * np.cos(grid)) ** 2 + (yt - a * dprev * np.sin(grid)) ** 2
        assert _angle_diff(al, grid[np.argmin(cost)]) <= 1e-3


def test_d_step_equals_1d_grid_minimiser():
    """d = argmin_{d >= 1} of Eq. 22a at the returned alpha, any (a, b), both rules."""
    rng = np.random.default_rng(1)
    for _ in range(300):
        xt, yt = rng.uniform(-4, 4, 2)
        a, b = rng.uniform(0.2, 2.0, 2)
        rule = int(rng.integers(0, 2))
        al, d = oracle.project_obstacle(xt, yt, a, b, rule)
        ca, sa = np.cos(al), np.sin(al)
        f = lambda dd: (xt - a * dd * ca) ** 2 + (yt - b * dd * sa) ** 2
        ds = np.linspace(1.0, 100.0, 990001)
        k = np.argmin(f(ds))
        lo, hi = ds[max(k - 1, 0)], ds[min(k + 1, ds.size - 1)]
        for _ in range(60):   # golden-section refinement inside the bracket
            m1, m2 = lo + 0.382 * (hi - lo), lo + 0.618 * (hi - lo)
            if f(m1) < f(m2):
                hi = m2
            else:
                lo = m1
        assert abs(d - 0.5 * (lo + hi)) <= 1e-6


def test_joint_projection_is_disk_exterior_projection():
    """For a = b the (alpha, d >= 1) step returns the nearest point of the disk exterior."""
    rng = np.random.default_rng(2)
    for _ in range(300):
        xt, yt = rng.uniform(-2, 2, 2)
        a = rng.uniform(0.3, 1.2)
        al, d = oracle.project_obstacle(xt, yt, a, a, 0)
        off = np.array([a * d * np.cos(al), a * d * np.sin(al)])
        rho_ = np.hypot(xt, yt)
        expect = np.array([xt, yt]) if rho_ >= a else a * np.array([xt, yt]) / rho_
        assert np.allclose(off, expect, atol=1e-12)


def test_scaled_rule_zero_residual_outside_ellipse():
    rng = np.random.default_rng(4)
    n_out = 0
    for _ in range(400):
        xt, yt = rng.uniform(-5, 5, 2)
        a, b = rng.uniform(0.3, 2.0, 2)
        al, d = oracle.project_obstacle(xt, yt, a, b, 1)
        if (xt / a) ** 2 + (yt / b) ** 2 >= 1.0:
            n_out += 1
            assert np.allclose([a * d * np.cos(al), b * d * np.sin(al)], [xt, yt], atol=1e-10)
    assert n_out > 100


def test_bound_projection_is_disk_projection():
    """Eq. 21b-22b with [0,1] clip (G6, G7): g_v = projection of v onto the v_max disk."""
    rng = np.random.default_rng(5)
    grid_a = np.linspace(-np.pi, np.pi, 721)
    grid_d = np.linspace(0.0, 1.0, 401)
    for _ in range(60):
        vx, vy = rng.uniform(-3, 3, 2)
        bound = rng.uniform(0.5, 2.5)
        al, d = oracle.project_bound(vx, vy, bound)
        g = d * bound * np.array([np.cos(al), np.sin(al)])
        v = np.array([vx, vy])
        nv_ = np.linalg.norm(v)
        assert np.allclose(g, v * min(1.0, bound / nv_), atol=1e-12)
        # brute force over the joint (alpha, d in [0, 1]) grid: no grid point is closer
        A, D = np.meshgrid(grid_a, grid_d)
        dist = (vx - D * bound * np.cos(A)) ** 2 + (vy - D * bound * np.sin(A)) ** 2
        assert np.sum((v - g) ** 2) <= dist.min() + 1e-12


@pytest.fixture(scope="module")
def scene():
    cfg = CONFIGS["C3"].with_(n=5, q=40)
    pr = make_problem(cfg, 2, B=3)
    o = Oracle(oracle_params(cfg), cfg.n)
    tr = o.trace_instance(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"][1], 6)
    return cfg, pr, o, tr


def test_lambda_step_is_fd_gradient(scene):
    """Eq. 23a (G3): Delta lambda = -rho grad_xi 0.5||F xi - g||^2."""
    cfg, pr, o, tr = scene
    xi, g = tr["xi1"][4], tr["g"][4]
    lam = tr["lam"][3][:44]
    new = o.lambda_step(lam, xi, g)
    h = 1e-6
    grad = np.zeros(44)
    for k in range(44):
        e = np.zeros(44)
        e[k] = h
        grad[k] = (o.penalty(xi + e, g) - o.penalty(xi - e, g)) / (2 * h)
    assert np.allclose((lam - new) / cfg.rho, grad, rtol=1e-5, atol=1e-6 * np.abs(grad).max())
    assert np.allclose(o.lambda_step(lam, xi, o.F @ xi), lam, atol=1e-12)


def test_trace_lambda_consistent_with_step(scene):
    cfg, pr, o, tr = scene
    for k in range(1, 6):
        new = o.lambda_step(tr["lam"][k - 1][:44], tr["xi1"][k], tr["g"][k])
        assert np.allclose(new, tr["lam"][k][:44], atol=1e-10)


def test_residual_pointwise(scene):
    """r1 equals the pointwise Eq. 7c-7g violation norm (rows rebuilt from BPoly)."""
    cfg, pr, o, tr = scene
    K = 5
    xi, g = tr["xi1"][K], tr["g"][K]
    t = np.linspace(0, cfg.T, cfg.q)
    q, m, n = cfg.q, cfg.m, cfg.n
    R = o.rows // 2
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
    assert abs(np.sqrt(tot) - tr["r1"][K]) <= 1e-10 * max(1.0, tr["r1"][K])
    psi = eval_bpoly(tr["xi2"][K], cfg.T, t)
    assert abs(np.linalg.norm(tr["theta"][K] - psi) - tr["rpsi"][K]) <= 1e-10


def test_boundary_holds_every_iteration(scene):
    """Boundary equalities to 1e-9 at every iterate (BASELINE north_star)."""
    cfg, pr, o, tr = scene
    t = np.array([0.0, cfg.T])
    for k in range(1, tr["xi1"].shape[0]):
        xi, xi2 = tr["xi1"][k], tr["xi2"][k]
        for ch, c in enumerate((xi[:11], xi[22:33], xi2)):
            vals = [eval_bpoly(c, cfg.T, t, nu) for nu in (0, 1, 2)]
            got = np.array([vals[0][0], vals[1][0], vals[2][0], vals[0][1], vals[1][1], vals[2][1]])
            assert np.max(np.abs(got - pr["bnd"][ch])) < 1e-9


def test_g_rows_are_geometric_projections(scene):
    """g (Eq. 10-11) rebuilt geometrically for circular obstacles: velocity/acceleration rows are
    the projections onto the v_max / a_max disks, collision rows the nearest point of the
    inflated obstacle's exterior to the circle centre (cos/sin psi, G9), copy rows cos/sin psi."""
    cfg, pr, o, tr = scene
    K = 4
    xi, xi2, g = tr["xi1"][K], tr["xi2"][K], tr["g"][K]
    t = np.linspace(0, cfg.T, cfg.q)
    q, m, n = cfg.q, cfg.m, cfg.n
    R = o.rows // 2
    x, xd, xdd = (eval_bpoly(xi[:11], cfg.T, t, nu) for nu in (0, 1, 2))
    y, yd, ydd = (eval_bpoly(xi[22:33], cfg.T, t, nu) for nu in (0, 1, 2))
    psi = eval_bpoly(xi2, cfg.T, t)

    def disk(vx, vy, bound):
        nrm = np.hypot(vx, vy)
        s = np.minimum(1.0, bound / np.maximum(nrm, 1e-300))
        return vx * s, vy * s

    gv = disk(xd, yd, cfg.v_max)
    ga = disk(xdd, ydd, cfg.a_max)
    assert np.allclose(g[:q], gv[0], atol=1e-10) and np.allclose(g[R:R + q], gv[1], atol=1e-10)
    assert np.allclose(g[q:2 * q], ga[0], atol=1e-10) and np.allclose(g[R + q:R + 2 * q], ga[1], atol=1e-10)
    obs = pr["obs_xy"].astype(np.float64)
    a = float(pr["obs_ab"][0, 0])
    for j in range(n):
        for i in range(m):
            cx = x + cfg.offsets[i] * np.cos(psi)
            cy = y + cfg.offsets[i] * np.sin(psi)
            dx, dy = cx - obs[j, 0], cy - obs[j, 1]
            dist = np.hypot(dx, dy)
            scale = np.maximum(1.0, a / dist)
            r0 = 2 * q + (j * m + i) * q
            assert np.allclose(g[r0:r0 + q], obs[j, 0] + dx * scale, atol=1e-9)
            assert np.allclose(g[R + r0:R + r0 + q], obs[j, 1] + dy * scale, atol=1e-9)
    assert np.allclose(g[2 * q + m * n * q:R], np.cos(psi), atol=1e-12)
    assert np.allclose(g[R + 2 * q + m * n * q:], np.sin(psi), atol=1e-12)


def test_iteration_wiring_on_a_cluttered_scene(scene):
    """Every iterate of a cluttered scene (5 obstacles, 3 circles) is the composition of
    the separately pinned steps in the paper's order (Algorithm of): xi1^{k+1}
    from (lambda^k, g^k) (Eq. 13, pinned by KKT optimality), theta^{k+1} = atan2 of the
    copies of xi1^{k+1} evaluated with the scipy BPoly basis (Eq. 19), xi2^{k+1} from
    (lambda_psi^k, theta^{k+1}) (Eq. 18, pinned by KKT optimality), g^{k+1} from the
    trajectory of (xi1^{k+1}, xi2^{k+1}) (test_g_rows_are_geometric_projections),
    lambda^{k+1} (test_trace_lambda_consistent_with_step) and lambda_psi^{k+1} =
    lambda_psi^k - rho_psi P^T (P xi2^{k+1} - theta^{k+1}) with the BPoly basis (Eq. 23b,
    G4).  A loop that fed a stale iterate to any step fails here."""
    cfg, pr, o, tr = scene
    t = np.linspace(0, cfg.T, cfg.q)
    P = np.stack([eval_bpoly(np.eye(11)[k], cfg.T, t) for k in range(11)], axis=1)   # q x 11
    bnd = pr["bnd"]
    for k in range(tr["xi1"].shape[0] - 1):
        lam, lampsi = tr["lam"][k][:44], tr["lam"][k][44:]
        xi1 = o.xi1_step(lam, tr["g"][k], bnd)
        assert np.allclose(xi1, tr["xi1"][k + 1], rtol=0, atol=1e-9 * max(1.0, np.abs(xi1).max())), k
        cc, ss = P @ xi1[11:22], P @ xi1[33:44]
        theta = np.arctan2(ss, cc)
        assert np.allclose(theta, tr["theta"][k + 1], atol=1e-10), k
        xi2 = o.xi2_step(lampsi, theta, bnd)
        assert np.allclose(xi2, tr["xi2"][k + 1], atol=1e-9), k
        lampsi_next = lampsi - cfg.rho_psi * (P.T @ (P @ xi2 - theta))
        assert np.allclose(lampsi_next, tr["lam"][k + 1][44:], atol=1e-9 * max(1.0, np.abs(lampsi_next).max())), k
