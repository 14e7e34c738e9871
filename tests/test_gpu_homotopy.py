"""NEXT-3: the method's quality claims as checks on synthetic scenes, solved on
the GPU at the operating point (B = 1000 Gaussian samples, K = 100) with the oracle
cross-checking a sample of each batch.

* Fig. 1c: one blocker on the straight line -> feasible trajectories in both
  homotopy classes (passing above and below);
* Table II trend: a wall with a 1.2 m gap -> the three-circle footprint passes
  through the gap, the conservative single disk covering the same 1.6 x 0.6 m footprint
  (radius 0.8 m) cannot and detours, so its best feasible trajectory is longer.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import Oracle  # noqa: E402
from synth import CONFIGS, make_init, scene_blocker, scene_wall_gap  # noqa: E402
from tests.helpers import bpoly_basis, oracle_params  # noqa: E402
from tests.parity import compare  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def solve(cfg, sc, init):
    from paper_2109_13030_b200 import solver_for
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out = solver_for(cfg, device=0).solve(d(init), d(sc["obs_xy"]), d(sc["obs_ab"]), sc["bnd"], cfg.K)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def geometry(cfg, coeffs):
    P, Pd, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    c = np.asarray(coeffs, np.float64)
    X, Y = P @ c[:, 0].T, P @ c[:, 2].T
    sp = np.hypot(Pd @ c[:, 0].T, Pd @ c[:, 2].T)
    dt = cfg.T / (cfg.q - 1)
    arc = (sp.sum(0) - 0.5 * (sp[0] + sp[-1])) * dt          # trapezoid rule
    return X, Y, arc


def y_at_x(X, Y, x0):
    i = np.argmin(np.abs(X - x0), axis=0)
    return Y[i, np.arange(X.shape[1])]


def oracle_check(cfg, sc, init, g, idx):
    o = Oracle(oracle_params(cfg), cfg.n)
    ref = o.solve(sc["bnd"], sc["obs_xy"], sc["obs_ab"], init[idx], cfg.K)
    gs = {k: g[k][idx] for k in ("coeffs", "lambda_out", "cost", "residual")}
    problem = dict(sc, init=init[idx])
    compare(cfg, gs, ref, cfg.res_tol, f"{cfg.name} sample", check_best=False, oracle=o, problem=problem)


def test_both_homotopies_around_a_blocker():
    sc = scene_blocker(100)
    cfg = CONFIGS["C3"].with_(name="blocker", n=1)
    init = make_init(cfg, seed=6, B=1000, sigma_y=5.0)
    g = solve(cfg, sc, init)
    X, Y, _ = geometry(cfg, g["coeffs"])
    feas = g["residual"][:, 0] <= cfg.res_tol
    side = np.sign(y_at_x(X, Y, 15.0))
    above, below = np.sum(feas & (side > 0)), np.sum(feas & (side < 0))
    assert feas.sum() > 300
    assert above > 0.05 * feas.sum() and below > 0.05 * feas.sum(), (above, below)
    # not instance 0: the unperturbed line meets the symmetric saddle exactly (y = 0 on both
    # sides of the obstacle), where either homotopy is an answer
    oracle_check(cfg, sc, init, g, np.arange(1, 1000, 125))


def test_multi_circle_passes_the_gap_single_disk_detours():
    res = {}
    for m, inflate in ((3, 0.3), (1, 0.8)):
        sc = scene_wall_gap(100, inflate=inflate)
        cfg = CONFIGS["C3"].with_(name=f"wall m={m}", m=m, n=sc["obs_xy"].shape[0])
        init = make_init(cfg, seed=5, B=1000, sigma_y=5.0)
        g = solve(cfg, sc, init)
        X, Y, arc = geometry(cfg, g["coeffs"])
        feas = g["residual"][:, 0] <= cfg.res_tol
        assert feas.any()
        best = int(g["best"][0])
        assert feas[best]
        res[m] = (arc[best], y_at_x(X, Y, 15.0)[best])
        # every footprint against the oracle (not instance 0: see above); the best
        # instance of each footprint is among the checked ones
        oracle_check(cfg, sc, init, g, np.unique(np.append(np.arange(1, 1000, 125), best if best else 1)))
    (arc3, y3), (arc1, y1) = res[3], res[1]
    assert abs(y3) < 0.35                      # three circles: through the gap
    assert abs(y1) > 3.3                       # single disk: around the wall
    assert arc3 < 0.97 * arc1, res
