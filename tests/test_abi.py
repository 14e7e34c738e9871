"""C-ABI library loads and exports every symbol include/bmc.h declares; parameter
validation paths that return before touching a device (no compute without a GPU)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bmc.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int32_t|void|const char\*)\s+(bmc_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2109_13030_b200 import load_library
    return load_library()


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("bmc_setup", "bmc_solve", "bmc_solve_host", "bmc_destroy", "bmc_last_error", "bmc_version",
              "bmc_last_launch_count", "bmc_sample_init", "bmc_pack_best", "bmc_select_best", "bmc_team_for"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    raw = C.CDLL(os.path.join(ROOT, "paper_2109_13030_b200", "libbmc.so"))
    for n in _declared():
        assert hasattr(raw, n), n
    assert lib.bmc_version() == 102


def _params(**kw):
    from paper_2109_13030_b200.bmc import BmcParams
    r = np.array(kw.pop("r", [-0.5, 0.0, 0.5]), dtype=np.float64)
    d = dict(q=100, T=30.0, degree=10, m=len(r), v_max=2.0, a_max=2.0, rho=1.0, rho_psi=1.0, w_copy=0.0,
             boundary_mask=0x3F, alpha_rule=0, res_tol=0.05, device=0)
    d.update(kw)
    p = BmcParams(d["q"], d["T"], d["degree"], d["m"], r.ctypes.data_as(C.POINTER(C.c_double)), d["v_max"],
                  d["a_max"], d["rho"], d["rho_psi"], d["w_copy"], d["boundary_mask"], d["alpha_rule"],
                  d["res_tol"], d["device"])
    return p, r


@pytest.mark.parametrize("kw,frag", [
    (dict(q=5), "q < degree"), (dict(q=200), "q > 128"), (dict(degree=7), "degree"),
    (dict(T=0.0), "T must"), (dict(m=0), "m must"), (dict(m=9), "m must"), (dict(v_max=0.0), "v_max"),
    (dict(rho=-1.0), "rho"), (dict(w_copy=-1.0), "w_copy"), (dict(boundary_mask=0x40), "boundary_mask"),
    (dict(alpha_rule=2), "alpha_rule"),
])
def test_setup_validation_without_device(lib, kw, frag):
    p, _r = _params(**kw)
    h = C.c_void_p()
    rc = lib.bmc_setup(C.byref(p), C.byref(h))
    assert rc == 1 and not h.value
    assert frag in lib.bmc_last_error().decode()


def test_setup_null_arguments(lib):
    h = C.c_void_p()
    assert lib.bmc_setup(None, C.byref(h)) == 1
    assert lib.bmc_solve(None, None, None, None) == 1
    assert lib.bmc_solve_host(None, None, None) == 1
    assert lib.bmc_team_for(None, 1000) == 0
    lib.bmc_destroy(None)


def test_exchange_entry_points_report_errors(lib):
    """bmc_pack_best / bmc_select_best validate before launching and set bmc_last_error."""
    lib.bmc_last_error()
    assert lib.bmc_pack_best(None, None, None, None, 0, None, None) == 1
    assert "bmc_pack_best" in lib.bmc_last_error().decode()
    buf = (C.c_int64 * 64)()
    assert lib.bmc_select_best(buf, 0, buf, buf, None) == 1
    assert "nranks" in lib.bmc_last_error().decode()


def test_setup_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p, _r = _params()
    h = C.c_void_p()
    rc = lib.bmc_setup(C.byref(p), C.byref(h))
    assert rc in (1, 3) and not h.value
