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
