"""The Python binding reuses its ctypes argument structs while the same buffer
objects come back (paper_2109_13030_b200/bmc.py Solver._marshal).  Host-only
check of the cache rule: identity of every buffer, equal scalars and boundary
values hit; anything else rebuilds."""
import numpy as np

from paper_2109_13030_b200.bmc import Solver


def _solver():
    s = Solver.__new__(Solver)   # no device: only the marshalling cache is exercised
    s._cache = {}
    return s


def test_cache_hits_only_for_identical_buffers_and_values():
    s = _solver()
    a, b = np.zeros(4, np.float32), np.zeros(4, np.float32)
    bnd = np.zeros((3, 6))
    calls = []

    def build():
        calls.append(1)
        return object(), object()

    first = s._marshal("host", (a, b, None), (10, 2, 5, 0), bnd, build)
    assert s._marshal("host", (a, b, None), (10, 2, 5, 0), bnd.copy(), build) is first   # equal values
    assert len(calls) == 1
    b2 = b.copy()                                                    # same contents, other buffer
    assert s._marshal("host", (a, b2, None), (10, 2, 5, 0), bnd, build) is not first
    assert s._marshal("host", (a, b2, None), (10, 2, 6, 0), bnd, build) is not None    # other iters
    bnd2 = bnd.copy()
    bnd2[0, 3] = 30.0
    n_before = len(calls)
    s._marshal("host", (a, b2, None), (10, 2, 6, 0), bnd2, build)                       # other boundary
    assert len(calls) == n_before + 1
    s._marshal("dev", (a, b2, None), (10, 2, 6, 0), bnd2, build)                        # other entry point
    assert len(calls) == n_before + 2


def test_problem_struct_carries_the_boundary_values():
    s = _solver()
    bnd = np.arange(18, dtype=np.float64).reshape(3, 6)
    p = s._problem(7, 3, 11, bnd, None, None, np.zeros((7, 3, 11), np.float32), None, 5)
    assert list(p.bnd) == list(range(18)) and p.B == 7 and p.n_obs == 3 and p.iters == 11 and p.index_base == 5
