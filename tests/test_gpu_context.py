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


def test_host_and_device_solves_from_two_threads():
    """bmc_solve (one thread, its own stream) and bmc_solve_host (another thread) on ONE
    context at the same time, with obstacle counts first seen by either path (so a blob
    uploaded on one stream is used by the other): every result is bitwise that of a
    fresh context solving alone (include/bmc.h "Threading / streams")."""
    import threading
    from paper_2109_13030_b200 import solver_for
    base = CONFIGS["C2"].with_(B=37, K=20)
    cases = {n: (base.with_(n=n), make_problem(base.with_(n=n), 50 + n)) for n in (5, 7, 9, 13)}
    ref = {n: _solve(solver_for(cfg, device=0), cfg, pr) for n, (cfg, pr) in cases.items()}
    shared = solver_for(base.with_(n=5), device=0)
    errors, got_dev, got_host = [], [], []

    def device_loop():
        try:
            st = torch.cuda.Stream()
            for n in (7, 5, 13, 7, 9, 5):
                cfg, pr = cases[n]
                with torch.cuda.stream(st):
                    got_dev.append((n, _solve(shared, cfg, pr, stream=st)))
        except Exception as e:   # pragma: no cover - reported below
            errors.append(e)

    def host_loop():
        try:
            for n in (9, 13, 5, 7, 9, 13):
                cfg, pr = cases[n]
                got_host.append((n, shared.solve_host(pr["init"], pr["obs_xy"], pr["obs_ab"], pr["bnd"], cfg.K)))
        except Exception as e:   # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=device_loop), threading.Thread(target=host_loop)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    assert len(got_dev) == 6 and len(got_host) == 6
    for n, g in got_dev + got_host:
        for k in ("coeffs", "lambda_out", "residual", "cost", "best"):
            assert np.array_equal(g[k], ref[n][k]), (n, k)


def test_solve_captured_in_a_cuda_graph():
    """After one warm-up solve (constants uploaded, shared-memory opt-in set), a solve is
    stream-ordered work only: captured into a CUDA graph and replayed, it writes the same
    bits as a direct solve, batch argmin included (the last CTA resets the workspace)."""
    from paper_2109_13030_b200 import solver_for
    cfg = CONFIGS["C2"].with_(B=64, K=12)
    pr = make_problem(cfg, 7)
    s = solver_for(cfg, device=0)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    init, obs, ab = d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"])
    ref = s.solve(init, obs, ab, pr["bnd"], cfg.K)
    torch.cuda.synchronize()
    ref = {k: v.clone() for k, v in ref.items()}
    out = {k: torch.empty_like(v) for k, v in ref.items()}
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):   # warm-up on the capture stream
        s.solve(init, obs, ab, pr["bnd"], cfg.K, out=out, stream=side)
    torch.cuda.synchronize()
    for v in out.values():
        v.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        s.solve(init, obs, ab, pr["bnd"], cfg.K, out=out, stream=torch.cuda.current_stream())
    assert s.last_launches == 1
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        for k in ref:
            assert torch.equal(out[k], ref[k]), k
