"""NEXT-2 on the GPU: bmc_sample_init against the oracle sampler
(oracle/sampler.c: same Philox4x32-10 stream, fp64 Box-Muller and STOMP factor), element by
element at fp32 rounding, the batch-split independence, and the error paths."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from synth import CONFIGS  # noqa: E402

pytestmark = pytest.mark.gpu

BND = np.array([[0.5, 1.0, 0.0, 30.0, 1.0, 0.0], [-1.0, 0.0, 0.0, 2.0, 0.0, 0.0], [0.0] * 6])


@pytest.fixture(scope="module")
def solver():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)
    from paper_2109_13030_b200 import solver_for
    return solver_for(CONFIGS["C3"], device=0)


@pytest.mark.parametrize("B,seed,stream,base", [(1, 1, 0, 0), (257, 7, 3, 0), (1000, 123456789012, 2**40 + 5, 77)])
def test_matches_oracle(solver, B, seed, stream, base):
    g = solver.sample_init(B, BND, seed, stream, sigma_x=1.0, sigma_y=5.0, index_base=base).cpu().numpy()
    ref = oracle.sample_init(B, BND, seed, stream, sigma_x=1.0, sigma_y=5.0, index_base=base)
    assert np.abs(g - ref).max() <= 4e-6 * (1.0 + np.abs(ref).max())
    # the x / y end control points are the segment's, fp32-rounded exactly once
    assert np.array_equal(g[:, 0, 0], np.full(B, np.float32(0.5)))


def test_split_independent_and_line_first(solver):
    full = solver.sample_init(300, BND, 5, 9).cpu().numpy()
    tail = solver.sample_init(200, BND, 5, 9, index_base=100).cpu().numpy()
    assert np.array_equal(full[100:], tail)
    k = np.arange(11) / 10
    assert np.allclose(full[0, 0], 0.5 + 29.5 * k) and np.allclose(full[0, 1], -1.0 + 3.0 * k)
    nol = solver.sample_init(4, BND, 5, 9, line_first=False).cpu().numpy()
    assert not np.allclose(nol[0, 1], full[0, 1])


def test_errors(solver):
    from paper_2109_13030_b200.bmc import BmcError
    assert solver.sample_init(0, BND, 1).shape[0] == 0
    bad = BND.copy()
    bad[0, 3] = np.nan
    with pytest.raises(BmcError):
        solver.sample_init(4, bad, 1)
