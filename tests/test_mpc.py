"""NEXT-1: the receding-horizon MPC loop (paper_2109_13030_b200/mpc.py)
driven by the fp64 oracle on CPU: host logic of the loop (boundary from the executed state,
warm-started multipliers, the executed state from the best trajectory), plus the Bernstein
evaluation helper against scipy."""
import numpy as np
import pytest

import oracle
from oracle import Oracle
from paper_2109_13030_b200.mpc import MPC, MPCConfig, bernstein_rows
from synth import CONFIGS, make_tracks
from tests.helpers import eval_bpoly, oracle_params


def test_bernstein_rows_match_bpoly():
    rng = np.random.default_rng(0)
    c = rng.standard_normal(11)
    for T in (10.0, 30.0):
        for t in (0.0, 0.1, 3.7, T):
            rows = bernstein_rows(10, t / T, T)
            for nu in range(3):
                assert abs(rows[nu] @ c - eval_bpoly(c, T, np.array([t]), nu)[0]) < 1e-11 * (1 + abs(c).sum())


class OracleBackend:
    """The MPC backend protocol on the fp64 oracle; records every call."""

    def __init__(self, cfg):
        self.o = Oracle(oracle_params(cfg), cfg.n)
        self.calls = []

    def sample(self, B, bnd, seed, stream, sigma_x, sigma_y):   # the oracle's STOMP sampler (NEXT-2)
        return oracle.sample_init(B, bnd, seed, stream, sigma_x=sigma_x, sigma_y=sigma_y).astype(np.float32)

    def __call__(self, init, obs_xy, obs_ab, bnd, K, lam):
        out = self.o.solve(bnd, obs_xy, obs_ab, init, K, lambda_in=lam)
        b = out["best_index"]
        self.calls.append(dict(init=init, obs_xy=obs_xy, obs_ab=obs_ab, bnd=bnd.copy(), lam=lam, out=out))
        return dict(lambda_out=out["lambda_out"], best=b, best_coeffs=out["coeffs"][b],
                    best_residual=out["residual"][b], best_cost=out["cost"][b])


def small_mpc(ticks=4, B=8):
    cfg = CONFIGS["C2"].with_(q=50, n=6)
    mc = MPCConfig(cfg, horizon=10.0, dt=0.2, K=10, seed=1)
    be = OracleBackend(mc.solve_cfg)
    m = MPC(mc, make_tracks(cfg, 1), be, B=B)
    for _ in range(ticks):
        m.tick()
    return mc, m, be


def test_mpc_loop_host_logic():
    mc, m, be = small_mpc()
    T = mc.horizon
    assert len(be.calls) == 4
    assert be.calls[0]["lam"] is None                        # cold start
    for k in range(1, 4):                                     # warm start: lambda_in = previous lambda_out
        assert be.calls[k]["lam"] is be.calls[k - 1]["out"]["lambda_out"]
    for k, r in enumerate(m.log):
        call = be.calls[k]
        c = r.coeffs
        # the best trajectory honours this tick's boundary (solver) ...
        for ch, blk in ((0, 0), (1, 2), (2, 4)):
            for nu in range(3):
                assert abs(eval_bpoly(c[blk], T, np.array([0.0]), nu)[0] - call["bnd"][ch, nu]) < 1e-6
        # ... and the executed state is that trajectory at t = dt (independent scipy evaluation)
        for ch, blk in ((0, 0), (1, 2), (2, 4)):
            for nu in range(3):
                assert abs(eval_bpoly(c[blk], T, np.array([mc.dt]), nu)[0] - r.state[ch, nu]) < 1e-9
        # next tick starts from it, and the goal recedes along the desired line
        if k + 1 < len(be.calls):
            nb = be.calls[k + 1]["bnd"]
            assert np.allclose(nb[:, 0:3], r.state)
            assert nb[0, 3] == pytest.approx(mc.v_des * (r.t + T))
    # the robot advances along +x at about v_des
    assert m.state[0, 0] == pytest.approx(mc.v_des * m.t, abs=0.2)


def test_mpc_obstacles_recede_with_time():
    mc, m, be = small_mpc(ticks=2)
    o0, o1 = be.calls[0]["obs_xy"], be.calls[1]["obs_xy"]
    tr = make_tracks(mc.cfg, 1)
    # the second tick sees every obstacle dt later along its track
    assert np.allclose(o1[:, 0, 0], (tr["x0"] + tr["vx"] * mc.dt).astype(np.float32))
    # and every sample moved by v dt
    assert np.allclose(o1[:, 0, :] - o0[:, 0, :], (tr["vx"] * mc.dt)[:, None], atol=1e-5)
    assert np.allclose(o1[:, 1, :] - o0[:, 1, :], (tr["vy"] * mc.dt)[:, None], atol=1e-5)
