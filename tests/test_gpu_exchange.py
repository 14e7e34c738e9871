"""Device side of the multi-GPU exchange (bmc_pack_best / bmc_select_best) on one GPU:
records packed from real shard solves, gathered by hand, and the selection must equal
the argmin over the concatenated batch."""
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


def test_pack_select_equals_global_argmin():
    import ctypes as C
    from paper_2109_13030_b200 import solver_for
    from paper_2109_13030_b200.bmc import load_library
    from paper_2109_13030_b200.distributed import RECORD_WORDS

    cfg = CONFIGS["C2"].with_(K=25)
    world, B = 3, 24
    pr = make_problem(cfg, 1, B=world * B)
    dev = torch.device("cuda", 0)
    s = solver_for(cfg, device=0)
    obs, ab = torch.from_numpy(pr["obs_xy"]).to(dev), torch.from_numpy(pr["obs_ab"]).to(dev)
    whole = s.solve(torch.from_numpy(pr["init"]).to(dev), obs, ab, pr["bnd"], cfg.K)
    records = torch.zeros(world * RECORD_WORDS, dtype=torch.int64, device=dev)
    L = load_library()
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    shard_outs = []
    for r in range(world):
        init = torch.from_numpy(np.ascontiguousarray(pr["init"][r * B:(r + 1) * B])).to(dev)
        o = s.solve(init, obs, ab, pr["bnd"], cfg.K, index_base=r * B)
        shard_outs.append(o)
        rec = records[r * RECORD_WORDS:(r + 1) * RECORD_WORDS]
        assert L.bmc_pack_best(C.c_void_p(o["best"].data_ptr()), C.c_void_p(o["coeffs"].data_ptr()),
                               C.c_void_p(o["residual"].data_ptr()), C.c_void_p(o["cost"].data_ptr()),
                               C.c_int64(r * B), C.c_void_p(rec.data_ptr()), stream) == 0
    best = torch.zeros(2, dtype=torch.int64, device=dev)
    coeffs = torch.zeros(55, dtype=torch.float32, device=dev)
    assert L.bmc_select_best(C.c_void_p(records.data_ptr()), 3, C.c_void_p(best.data_ptr()),
                             C.c_void_p(coeffs.data_ptr()), stream) == 0
    torch.cuda.synchronize()
    # shard solves are bitwise equal to the whole-batch rows (independent instances)
    for r, o in enumerate(shard_outs):
        assert torch.equal(o["coeffs"], whole["coeffs"][r * B:(r + 1) * B])
    assert int(best[0]) == int(whole["best"][0]) and int(best[1]) == int(whole["best"][1])
    assert torch.equal(coeffs, whole["coeffs"][int(best[0])].reshape(-1))
    # the winning record carries the instance's residuals and cost (floats 55..57)
    b = int(best[0])
    recs = records.view(world, RECORD_WORDS)
    win = recs[int(torch.argmin(recs[:, 0]))][1:].clone().view(torch.float32)
    assert torch.equal(win[55:57], whole["residual"][b]) and float(win[57]) == float(whole["cost"][b])


def test_sharded_entry_points_single_rank_nccl():
    """solve_sharded / solve_sharded_host over a one-rank NCCL group: the exchange
    reads the shard's best from device outputs and, on the host path, from
    page-locked host outputs mapped into the device address space."""
    import os
    import socket

    import torch.distributed as dist
    from paper_2109_13030_b200 import solver_for
    from paper_2109_13030_b200.distributed import BestExchange, solve_sharded, solve_sharded_host

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        cfg = CONFIGS["C2"].with_(B=40, K=20)
        pr = make_problem(cfg, 3)
        s = solver_for(cfg, device=0)
        x = BestExchange(dist.group.WORLD, dev)
        d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        out, best, coeffs = solve_sharded(s, x, d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], cfg.K,
                                          index_base=500)
        torch.cuda.synchronize()
        b = int(best[0])
        assert 500 <= b < 540 and int(best[1]) == int(out["best"][1])
        assert torch.equal(coeffs, out["coeffs"][b - 500].reshape(-1))
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        h = {k: pin(np.empty(tuple(v.shape), np.float32 if v.dtype == torch.float32 else np.int64))
             for k, v in out.items()}
        _, hb, hc = solve_sharded_host(s, x, pin(pr["init"]), pin(pr["obs_xy"]), pin(pr["obs_ab"]), pr["bnd"], cfg.K,
                                       500, out=h)
        assert np.array_equal(hb, best.cpu().numpy()) and np.array_equal(hc, coeffs.cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_c3_as_eight_shards_is_bitwise_the_one_gpu_solve():
    """The bench batch (C3, B = 1000) solved as 8 shards of 125 (what 8 GPUs run), with
    the team size of the whole batch (Solver.team_for): every instance is bitwise the
    one-GPU solve's, and the exchange over the 8 records (plus one empty shard, key ~0)
    returns the one-GPU global best.  With the automatic team of a 125-instance shard
    (4 warps per instance instead of 2) the fp64 partial sums are combined in another
    order; those shards still pick the same global best."""
    import ctypes as C
    from paper_2109_13030_b200 import solver_for
    from paper_2109_13030_b200.bmc import load_library
    from paper_2109_13030_b200.distributed import EMPTY_KEY, RECORD_WORDS

    cfg = CONFIGS["C3"]
    pr = make_problem(cfg, 0)
    dev = torch.device("cuda", 0)
    s = solver_for(cfg, device=0)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    obs, ab = d(pr["obs_xy"]), d(pr["obs_ab"])
    whole = s.solve(d(pr["init"]), obs, ab, pr["bnd"], cfg.K)
    team = s.team_for(cfg.B)
    assert team == 2 and s.team_for(125) == 4
    L = load_library()
    stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    world, per = 8, 125
    for team_arg in (team, 0):
        records = torch.zeros((world + 1) * RECORD_WORDS, dtype=torch.int64, device=dev)
        outs = []
        for r in range(world):
            o = s.solve(d(pr["init"][r * per:(r + 1) * per]), obs, ab, pr["bnd"], cfg.K, index_base=r * per,
                        team=team_arg)
            outs.append(o)
            rec = records[r * RECORD_WORDS:(r + 1) * RECORD_WORDS]
            assert L.bmc_pack_best(C.c_void_p(o["best"].data_ptr()), C.c_void_p(o["coeffs"].data_ptr()),
                                   None, None, C.c_int64(r * per), C.c_void_p(rec.data_ptr()), stream) == 0
        empty = torch.tensor([0, EMPTY_KEY], dtype=torch.int64, device=dev)
        rec = records[world * RECORD_WORDS:]
        assert L.bmc_pack_best(C.c_void_p(empty.data_ptr()), C.c_void_p(whole["coeffs"].data_ptr()),
                               None, None, C.c_int64(cfg.B), C.c_void_p(rec.data_ptr()), stream) == 0
        best = torch.zeros(2, dtype=torch.int64, device=dev)
        coeffs = torch.zeros(55, dtype=torch.float32, device=dev)
        assert L.bmc_select_best(C.c_void_p(records.data_ptr()), world + 1, C.c_void_p(best.data_ptr()),
                                 C.c_void_p(coeffs.data_ptr()), stream) == 0
        torch.cuda.synchronize()
        assert int(best[0]) == int(whole["best"][0])
        if team_arg:
            for r, o in enumerate(outs):
                for k in ("coeffs", "lambda_out", "residual", "cost"):
                    assert torch.equal(o[k], whole[k][r * per:(r + 1) * per]), (r, k)
            assert int(best[1]) == int(whole["best"][1])
            assert torch.equal(coeffs, whole["coeffs"][int(best[0])].reshape(-1))
