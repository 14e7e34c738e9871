"""NEXT-1 on the GPU: the MPC tick (warm-started multipliers, K = 10).

* tick-level parity: the oracle drives the loop; every tick's exact inputs (fresh samples,
  receding obstacles, boundary from the executed state, lambda_in = the previous tick's
  lambda_out) are replayed through the C-ABI and compared element by element;
* the GPU loop at the paper's operating point (B = 1000, K = 10): progress along the desired
  line and the per-tick device time against the paper's 0.04 s budget.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import Oracle  # noqa: E402
from synth import CONFIGS, make_tracks  # noqa: E402
from tests.helpers import oracle_params  # noqa: E402
from tests.parity import compare  # noqa: E402
from tests.test_mpc import small_mpc  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def test_mpc_ticks_match_oracle():
    from paper_2109_13030_b200 import solver_for
    mc, m, be = small_mpc(ticks=4, B=24)
    sc = mc.solve_cfg
    s = solver_for(sc, device=0)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.float32))).cuda()
    for k, call in enumerate(be.calls):
        lam = None if call["lam"] is None else d(call["lam"])
        out = s.solve(d(call["init"]), d(call["obs_xy"]), d(call["obs_ab"]), call["bnd"], mc.K, lambda_in=lam)
        torch.cuda.synchronize()
        g = {key: v.cpu().numpy() for key, v in out.items()}
        problem = dict(init=call["init"], obs_xy=call["obs_xy"], obs_ab=call["obs_ab"], bnd=call["bnd"])
        compare(sc, g, call["out"], sc.res_tol, f"MPC tick {k}", oracle=Oracle(oracle_params(sc), sc.n),
                problem=problem, iters=mc.K, lambda_in=call["lam"])


def test_mpc_loop_at_paper_operating_point():
    from paper_2109_13030_b200.mpc import MPC, GpuBackend, MPCConfig
    cfg = CONFIGS["C3"]
    mc = MPCConfig(cfg, horizon=10.0, dt=0.1, K=10, seed=2)
    m = MPC(mc, make_tracks(cfg, 2), GpuBackend(mc), B=1000)
    for _ in range(30):
        m.tick()
    ms = np.array([r.solve_ms for r in m.log[5:]])
    assert ms.max() < 40.0                                  # the paper's 0.04 s tick budget
    assert m.state[0, 0] > 0.8 * mc.v_des * m.t             # progress along the desired line
    assert np.all(np.isfinite([r.cost for r in m.log]))
