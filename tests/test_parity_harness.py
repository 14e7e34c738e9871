"""The GPU<->oracle comparison harness itself (CPU): the bar applies to every output
(x, y, psi, copies, cost, residuals, multipliers); a deviation beyond it passes only
on an instance where the oracle's own fp32 rounding model moves the answer as far
(within KAPPA); and the best index is checked for near-optimality on ambiguous
scenes.  Also the fp32 rounding model itself (oracle.h `fp32_model`)."""
import dataclasses

import numpy as np
import pytest

from oracle import Oracle
from synth import CONFIGS, make_problem
from tests.helpers import bpoly_basis, oracle_params
from tests.parity import KAPPA, compare, deviations


@pytest.fixture(scope="module")
def c2():
    cfg = CONFIGS["C2"]
    pr = make_problem(cfg, 0, B=37)
    o = Oracle(oracle_params(cfg), cfg.n)
    ref = o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K)
    return cfg, pr, o, ref


def _copy(ref):
    return {k: np.array(ref[k], copy=True) for k in ("coeffs", "lambda_out", "cost", "residual")}


def test_identical_results_pass(c2):
    cfg, pr, o, ref = c2
    g = dict(coeffs=ref["coeffs"].astype(np.float32), lambda_out=ref["lambda_out"].astype(np.float32),
             cost=ref["cost"], residual=ref["residual"], best=np.array([ref["best_index"], ref["best_key"]]))
    st = compare(cfg, g, ref, cfg.res_tol, "self")
    assert st["max_dtraj"] < 1e-5 and not st["fp32_model_accepted"]


@pytest.mark.parametrize("what", ["cost", "psi", "copy", "lambda", "r_psi"])
def test_rejects_deviation_on_well_conditioned_instance(c2, what):
    """Every output is under the bar: an error injected into any of them on a
    well-conditioned instance (fp32-model spread ~1e-6) is rejected."""
    cfg, pr, o, ref = c2
    g = _copy(ref)
    i = 3
    if what == "cost":
        g["cost"][i] *= 1 + 5e-4
    elif what == "psi":
        g["coeffs"][i, 4, 5] += 6e-3           # mid-horizon heading coefficient: 1.5e-3 rad
    elif what == "copy":
        g["coeffs"][i, 1, 5] += 6e-3
    elif what == "lambda":
        g["lambda_out"][i] *= 1 + 5e-3
    else:
        g["residual"][i, 1] += 1e-3 + 1e-3 * abs(g["residual"][i, 1])
    with pytest.raises(AssertionError):
        compare(cfg, g, ref, cfg.res_tol, f"injected {what}", check_best=False, oracle=o, problem=pr)


@pytest.fixture(scope="module")
def c3_sensitive():
    """C3 (seed 4) instances 2 and 8: #2 is infeasible (r1 ~ 1.15) and moves by 1e-4..5e-4 m
    under the fp32 rounding model; #8 barely moves."""
    cfg = CONFIGS["C3"]
    pr = make_problem(cfg, 4, B=40)
    sub = dict(pr, init=np.ascontiguousarray(pr["init"][[2, 8]]))
    o = Oracle(oracle_params(cfg), cfg.n)
    ref = o.solve(sub["bnd"], sub["obs_xy"], sub["obs_ab"], sub["init"], cfg.K)
    return cfg, sub, o, ref


def test_another_fp32_run_is_accepted_on_the_sensitive_instance(c3_sensitive):
    """A further fp32-model run (a seed the harness does not use) stands in for another
    fp32 implementation: on #2 it misses the plain bar and is accepted by the model
    spread; #8 meets the plain bar."""
    cfg, pr, o, ref = c3_sensitive
    om = Oracle(dataclasses.replace(o.params, fp32_model=1, noise_seed=977), o.n)
    g = om.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K)
    st = compare(cfg, g, ref, cfg.res_tol, "another fp32 run", check_best=False, oracle=o, problem=pr)
    assert [a["inst"] for a in st["fp32_model_accepted"]] in ([0], [])
    assert all(a["max_ratio"] <= KAPPA for a in st["fp32_model_accepted"])


def test_deviation_far_beyond_the_spread_is_rejected(c3_sensitive):
    cfg, pr, o, ref = c3_sensitive
    for inst, rel in ((0, 2e-2), (1, 3e-4)):
        g = _copy(ref)
        g["cost"][inst] *= 1 + rel
        with pytest.raises(AssertionError):
            compare(cfg, g, ref, cfg.res_tol, "far", check_best=False, oracle=o, problem=pr)


def test_best_index_near_optimality_on_ambiguous_scenes(c2):
    """A different best index passes only if the scene is ambiguous AND the oracle's value
    at the GPU's pick is within 1e-4 of the best; on an unambiguous scene it fails."""
    cfg, pr, o, ref = c2
    r1 = ref["residual"][:, 0]
    feas = r1 <= cfg.res_tol
    v = np.where(feas, ref["cost"], r1)
    order = np.lexsort((np.arange(len(v)), v, ~feas))
    g = _copy(ref)
    worst = int(order[-1])
    g["best"] = np.array([worst, 0])
    with pytest.raises(AssertionError):
        compare(cfg, g, ref, cfg.res_tol, "wrong best")
    # make the runner-up tie the best within 1e-5: ambiguous, and its pick is near-optimal
    ref2 = dict(ref, cost=np.array(ref["cost"], copy=True))
    b0, b1 = int(order[0]), int(order[1])
    if feas[b0] and feas[b1]:
        ref2["cost"][b1] = ref2["cost"][b0] * (1 + 1e-5)
        g2 = _copy(ref2)
        g2["best"] = np.array([b1, 0])
        compare(cfg, g2, ref2, cfg.res_tol, "ambiguous, near-optimal pick")
        ref3 = dict(ref2, cost=np.array(ref2["cost"], copy=True))
        ref3["cost"][b1] = ref3["cost"][b0] * (1 + 5e-4)     # ambiguous (1e-3) but beyond 1e-4
        g3 = _copy(ref3)
        g3["best"] = np.array([b1, 0])
        with pytest.raises(AssertionError):
            compare(cfg, g3, ref3, cfg.res_tol, "ambiguous, pick not near-optimal")


def test_fp32_model_round_to_nearest_is_close_on_well_conditioned_instances(c2):
    """The fp32 rounding model (round to nearest) stays within fp32-scale distance of the
    fp64 oracle on most instances, is deterministic, and seeds change its rounding."""
    cfg, pr, o, ref = c2
    P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
    m0 = Oracle(dataclasses.replace(o.params, fp32_model=1, noise_seed=0), o.n)
    a = m0.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K)
    b = m0.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K)
    assert np.array_equal(a["coeffs"], b["coeffs"])
    d = deviations(P, a, ref)
    assert np.median(d["traj"]) < 1e-5 and np.median(d["traj"]) > 0
    m1 = Oracle(dataclasses.replace(o.params, fp32_model=1, noise_seed=5), o.n)
    c = m1.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K)
    assert not np.array_equal(a["coeffs"], c["coeffs"])
    assert np.median(deviations(P, c, ref)["traj"]) < 1e-5
