"""fp64 CPU oracle of the batched AM iteration (arXiv 2109.13030).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_2109_13030_b200``) never imports it, and
the two share no code: this is a ctypes wrapper around ``oracle.c`` (plain C,
fp64, libm), which follows PAPER.md step by step (see oracle.c's header for
the equation map and the readings G1..G18).

Parity status per function:
  basis, KKT steps, projections, lambda and lambda_psi steps, cost J,
  obstacle-free fixed point, invariants, worked-scene residual decay: pinned by
  tests/test_oracle_*.py.  Iterates on cluttered scenes: the paper prints no
  worked iterate; they are pinned as the composition of the pinned steps in
  the paper's order (test_iteration_wiring_on_a_cluttered_scene: every
  iterate recomputed from its predecessor with the pinned steps and an
  independent BPoly basis) and through the invariants above.

fp32 rounding model (OracleParams.fp32_model / noise_seed, oracle.h): the same
iteration with every quantity the product path holds in fp32 rounded where it
is formed (stochastically when seeded).  It is a measuring instrument of the
parity harness (tests/parity.py): how far fp32 rounding alone moves an
instance.  Off by default; the fp64 path is unchanged by it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = C.POINTER(C.c_double)
_llp = C.POINTER(C.c_longlong)


class _Params(C.Structure):
    _fields_ = [
        ("q", C.c_int),
        ("T", C.c_double),
        ("degree", C.c_int),
        ("m", C.c_int),
        ("r", _dp),
        ("v_max", C.c_double),
        ("a_max", C.c_double),
        ("rho", C.c_double),
        ("rho_psi", C.c_double),
        ("w_copy", C.c_double),
        ("boundary_mask", C.c_uint),
        ("alpha_rule", C.c_int),
        ("lampsi_printed_sign", C.c_int),
        ("res_tol", C.c_double),
        ("fp32_model", C.c_int),
        ("noise_seed", C.c_ulonglong),
    ]


def build(force: bool = False) -> str:
    """Compile liboracle.so in place (gcc -O2 -fopenmp, no fast-math)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIBPATH) or os.path.getmtime(_LIBPATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "-B" if force else "liboracle.so"], check=True,
                       env={k: v for k, v in os.environ.items() if k != "CFLAGS"})
    return _LIBPATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIBPATH)
        L.or_basis.argtypes = [C.c_int, C.c_double, C.c_int, _dp, _dp, _dp]
        L.or_create.argtypes = [C.POINTER(_Params), C.c_int, C.POINTER(C.c_int)]
        L.or_create.restype = C.c_void_p
        L.or_destroy.argtypes = [C.c_void_p]
        for nm in ("or_nv", "or_nb", "or_rows"):
            getattr(L, nm).argtypes = [C.c_void_p]
            getattr(L, nm).restype = C.c_int
        for nm in ("or_F", "or_Qbar", "or_A", "or_kkt1", "or_kkt1_inv", "or_kktpsi",
                   "or_kktpsi_inv", "or_basis_P", "or_basis_Pd", "or_basis_Pdd"):
            getattr(L, nm).argtypes = [C.c_void_p]
            getattr(L, nm).restype = _dp
        L.or_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_longlong, _dp, _dp, _dp, _dp,
                               _dp, _dp, _dp, _dp, _dp, _dp, _llp, C.c_int]
        L.or_trace_instance.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                        _dp, _dp, _dp, _dp, _dp]
        L.or_project_obstacle.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
                                          _dp, _dp]
        L.or_project_bound.argtypes = [C.c_double, C.c_double, C.c_double, _dp, _dp]
        L.or_penalty.argtypes = [C.c_void_p, _dp, _dp]
        L.or_penalty.restype = C.c_double
        L.or_lambda_step.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        L.or_xi1_step.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        L.or_xi2_step.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        L.or_philox4x32_10.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.or_philox4x32_10.restype = None
        L.or_stomp_factor.argtypes = [C.c_int, _dp, C.POINTER(C.c_int)]
        L.or_stomp_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_longlong, _dp]
        L.or_stomp_normals.restype = None
        L.or_sample_init.argtypes = [C.c_int, C.c_longlong, C.c_longlong, C.c_uint64, C.c_uint64, _dp,
                                     C.c_double, C.c_double, C.c_int, _dp]
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous fp64"
    return a.ctypes.data_as(_dp)


def _f64(a) -> Optional[np.ndarray]:
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


@dataclass
class OracleParams:
    q: int
    T: float
    degree: int
    r: Sequence[float]
    v_max: float
    a_max: float
    rho: float = 1.0
    rho_psi: float = 1.0
    w_copy: float = 0.0
    boundary_mask: int = 0x3F
    alpha_rule: int = 0
    lampsi_printed_sign: int = 0
    res_tol: float = 1e-2
    fp32_model: int = 0          # parity harness: fp32 rounding model (oracle.h)
    noise_seed: int = 0          # 0: round to nearest; else stochastic rounding keyed by this seed
    _r: np.ndarray = field(default=None, repr=False)

    def to_c(self) -> _Params:
        self._r = _f64(self.r)
        return _Params(self.q, self.T, self.degree, len(self._r), _ptr(self._r), self.v_max,
                       self.a_max, self.rho, self.rho_psi, self.w_copy, self.boundary_mask,
                       self.alpha_rule, self.lampsi_printed_sign, self.res_tol, self.fp32_model,
                       self.noise_seed)


def basis(q: int, T: float, degree: int):
    nv = degree + 1
    P, Pd, Pdd = (np.zeros((q, nv)) for _ in range(3))
    rc = lib().or_basis(q, T, degree, _ptr(P), _ptr(Pd), _ptr(Pdd))
    if rc != 0:
        raise ValueError(f"or_basis failed: {rc}")
    return P, Pd, Pdd


def project_obstacle(xt: float, yt: float, a: float, b: float, rule: int = 0):
    al, d = C.c_double(), C.c_double()
    lib().or_project_obstacle(xt, yt, a, b, rule, C.byref(al), C.byref(d))
    return al.value, d.value


def project_bound(vx: float, vy: float, bound: float):
    al, d = C.c_double(), C.c_double()
    lib().or_project_bound(vx, vy, bound, C.byref(al), C.byref(d))
    return al.value, d.value


class Oracle:
    """Problem of Eq. 9-12 for a fixed obstacle count n (F, Q_bar, KKT inverses)."""

    def __init__(self, params: OracleParams, n_obs: int):
        self.params = params
        self.n = n_obs
        self._cp = params.to_c()
        err = C.c_int(0)
        self._h = lib().or_create(C.byref(self._cp), n_obs, C.byref(err))
        if not self._h:
            raise ValueError(f"or_create failed with code {err.value}")
        L = lib()
        self.nv = L.or_nv(self._h)
        self.nb = L.or_nb(self._h)
        self.rows = L.or_rows(self._h)
        self.q = params.q
        self.m = len(params.r)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_destroy(self._h)
            self._h = None

    def _mat(self, fn: str, shape):
        p = getattr(lib(), fn)(self._h)
        return np.ctypeslib.as_array(p, shape=shape).copy()

    @property
    def F(self):
        return self._mat("or_F", (self.rows, 4 * self.nv))

    @property
    def Qbar(self):
        return self._mat("or_Qbar", (4 * self.nv, 4 * self.nv))

    @property
    def A(self):
        return self._mat("or_A", (max(self.nb, 1), self.nv))[: self.nb]

    @property
    def kkt1(self):
        N = 4 * self.nv + 2 * self.nb
        return self._mat("or_kkt1", (N, N))

    @property
    def kkt1_inv(self):
        N = 4 * self.nv + 2 * self.nb
        return self._mat("or_kkt1_inv", (N, N))

    @property
    def kktpsi(self):
        N = self.nv + self.nb
        return self._mat("or_kktpsi", (N, N))

    @property
    def kktpsi_inv(self):
        N = self.nv + self.nb
        return self._mat("or_kktpsi_inv", (N, N))

    @property
    def P(self):
        return self._mat("or_basis_P", (self.q, self.nv))

    @property
    def Pd(self):
        return self._mat("or_basis_Pd", (self.q, self.nv))

    @property
    def Pdd(self):
        return self._mat("or_basis_Pdd", (self.q, self.nv))

    def solve(self, bnd, obs_xy, obs_ab, init, iters: int, lambda_in=None, trace: bool = False,
              index_base: int = 0, nthreads: int = 0) -> dict:
        init = _f64(init)
        B = init.shape[0]
        nv = self.nv
        bnd, obs_xy, obs_ab, lam_in = _f64(bnd), _f64(obs_xy), _f64(obs_ab), _f64(lambda_in)
        if self.n == 0:
            obs_xy = np.zeros((1, 2, self.q)) if obs_xy is None or obs_xy.size == 0 else obs_xy
            obs_ab = np.ones((1, 2)) if obs_ab is None or obs_ab.size == 0 else obs_ab
        coeffs = np.zeros((B, 5, nv))
        lam_out = np.zeros((B, 5, nv))
        residual = np.zeros((B, 2))
        cost = np.zeros(B)
        res_trace = np.zeros((B, iters)) if trace and iters > 0 else None
        best = np.zeros(2, dtype=np.int64)
        rc = lib().or_solve(self._h, B, iters, index_base, _ptr(bnd), _ptr(obs_xy), _ptr(obs_ab),
                            _ptr(init), _ptr(lam_in), _ptr(coeffs), _ptr(lam_out), _ptr(residual),
                            _ptr(cost), _ptr(res_trace), best.ctypes.data_as(_llp), nthreads)
        if rc != 0:
            raise ValueError(f"or_solve failed with code {rc}")
        out = dict(coeffs=coeffs, lambda_out=lam_out, residual=residual, cost=cost,
                   best_index=int(best[0]), best_key=int(best[1]))
        if res_trace is not None:
            out["res_trace"] = res_trace
        return out

    def trace_instance(self, bnd, obs_xy, obs_ab, init, iters: int, lambda_in=None) -> dict:
        nv, K, q = self.nv, iters, self.q
        init = _f64(init).reshape(3, nv)
        bnd, obs_xy, obs_ab, lam_in = _f64(bnd), _f64(obs_xy), _f64(obs_ab), _f64(lambda_in)
        if self.n == 0:
            obs_xy = np.zeros((1, 2, q))
            obs_ab = np.ones((1, 2))
        xi1 = np.zeros((K + 1, 4 * nv))
        xi2 = np.zeros((K + 1, nv))
        lam = np.zeros((K + 1, 5 * nv))
        g = np.zeros((K + 1, self.rows))
        theta = np.zeros((K + 1, q))
        r1 = np.zeros(K + 1)
        rpsi = np.zeros(K + 1)
        rc = lib().or_trace_instance(self._h, K, _ptr(bnd), _ptr(obs_xy), _ptr(obs_ab), _ptr(init),
                                     _ptr(lam_in), _ptr(xi1), _ptr(xi2), _ptr(lam), _ptr(g),
                                     _ptr(theta), _ptr(r1), _ptr(rpsi))
        if rc != 0:
            raise ValueError(f"or_trace_instance failed with code {rc}")
        return dict(xi1=xi1, xi2=xi2, lam=lam, g=g, theta=theta, r1=r1, rpsi=rpsi)

    def penalty(self, xi1, g) -> float:
        return lib().or_penalty(self._h, _ptr(_f64(xi1)), _ptr(_f64(g)))

    def lambda_step(self, lam, xi1, g):
        out = np.zeros(4 * self.nv)
        lib().or_lambda_step(self._h, _ptr(_f64(lam)), _ptr(_f64(xi1)), _ptr(_f64(g)), _ptr(out))
        return out

    def xi1_step(self, lam, g, bnd):
        out = np.zeros(4 * self.nv)
        lib().or_xi1_step(self._h, _ptr(_f64(lam)), _ptr(_f64(g)), _ptr(_f64(bnd)), _ptr(out))
        return out

    def xi2_step(self, lampsi, theta, bnd):
        out = np.zeros(self.nv)
        lib().or_xi2_step(self._h, _ptr(_f64(lampsi)), _ptr(_f64(theta)), _ptr(_f64(bnd)), _ptr(out))
        return out


# ---- STOMP-style initial samples (sampler.c) -------------------------

def philox4x32_10(ctr, key):
    """One Philox4x32-10 block: 4 x uint32 counter, 2 x uint32 key -> 4 x uint32."""
    c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (C.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return [int(v) for v in o]


def stomp_factor(degree: int = 10) -> np.ndarray:
    L = np.zeros(256)
    nf = C.c_int(0)
    rc = lib().or_stomp_factor(degree, _ptr(L), C.byref(nf))
    if rc != 0:
        raise ValueError(f"or_stomp_factor failed with code {rc}")
    return L[: nf.value * nf.value].reshape(nf.value, nf.value)


def stomp_normals(seed: int, stream: int, g: int) -> np.ndarray:
    z = np.zeros(12)
    lib().or_stomp_normals(seed, stream, g, _ptr(z))
    return z


def sample_init(B: int, bnd, seed: int, stream: int = 0, sigma_x: float = 1.0, sigma_y: float = 5.0,
                index_base: int = 0, line_first: bool = True, degree: int = 10) -> np.ndarray:
    """init [B][3][degree+1] fp64: straight segment p0 -> pT plus STOMP noise (reading G28)."""
    out = np.zeros((B, 3, degree + 1))
    rc = lib().or_sample_init(degree, B, index_base, seed, stream, _ptr(_f64(bnd)), sigma_x, sigma_y,
                              int(line_first), _ptr(out))
    if rc != 0:
        raise ValueError(f"or_sample_init failed with code {rc}")
    return out
