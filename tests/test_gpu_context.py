"""Context behaviour on the GPU: the per-n constant cache (bounded, least recently used
evicted) and its asynchronous upload on the solve's stream (include/bmc.h bmc_solve)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from synth import CONFIGS, make_problem  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def _solve(s, cfg, pr, stream=None):
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out = s.solve(d(pr["init"]), d(pr["obs_xy"]) if cfg.n else None, d(pr["obs_ab"]) if cfg.n else None,
                  pr["bnd"], cfg.K, stream=stream)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def test_constant_cache_eviction_and_async_upload():
    """Twelve obstacle counts on one context (more than the 8 it keeps), each first solved
    on a side stream right after its inputs were produced there: every result is bitwise
    that of a fresh context, also for counts solved again after their eviction."""
    from paper_2109_13030_b200 import solver_for
    base = CONFIGS["C2"].with_(B=24, K=15)
    shared = solver_for(base, device=0)
    side = torch.cuda.Stream()
    ns = list(range(0, 12)) + [0, 3, 11]
    for n in ns:
        cfg = base.with_(n=n)
        pr = make_problem(cfg, 20 + n)
        with torch.cuda.stream(side):
            got = _solve(shared, cfg, pr, stream=side)
        ref = _solve(solver_for(cfg, device=0), cfg, pr)
        for k in ("coeffs", "lambda_out", "residual", "cost", "best"):
            assert np.array_equal(got[k], ref[k]), (n, k)
