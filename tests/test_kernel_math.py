"""Host-side checks of closed forms the CUDA kernel relies on (no GPU needed).

* Bernstein derivative operator: Pdot = P Dm and Pddot = P Dm^2 with the tridiagonal
  Dm of bmc_kernel.cuh (dm_apply), against the independent scipy basis of tests/helpers.
* atan2_fast: the polynomial coefficients are parsed from bmc_kernel.cuh and evaluated
  in float32 (numpy) exactly as the kernel orders the operations; error bound and bias
  against numpy's arctan2 in fp64.
"""
import os
import re

import numpy as np
import pytest

from tests.helpers import bpoly_basis

KERNEL = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "paper_2109_13030_b200", "csrc", "bmc_kernel.cuh")


def dm_matrix(n, T):
    """(Dm c)_k = (-k c_{k-1} + (2k - n) c_k + (n - k) c_{k+1}) / T."""
    D = np.zeros((n + 1, n + 1))
    for k in range(n + 1):
        if k >= 1:
            D[k, k - 1] = -k / T
        D[k, k] = (2 * k - n) / T
        if k < n:
            D[k, k + 1] = (n - k) / T
    return D


@pytest.mark.parametrize("q,T", [(100, 30.0), (50, 12.5), (128, 7.0), (33, 1.0)])
def test_bernstein_derivative_operator(q, T):
    P, Pd, Pdd = bpoly_basis(q, T, 10)
    D = dm_matrix(10, T)
    assert np.abs(P @ D - Pd).max() <= 1e-12 * np.abs(Pd).max()
    assert np.abs(P @ D @ D - Pdd).max() <= 1e-12 * np.abs(Pdd).max()
    # the transposed use in the contraction: Pd^T u = Dm^T (P^T u)
    u = np.random.default_rng(0).standard_normal(q)
    assert np.allclose(Pd.T @ u, D.T @ (P.T @ u), rtol=1e-12, atol=1e-12 * np.abs(Pd.T @ u).max())


def _atan2_coeffs():
    src = open(KERNEL).read()
    body = src[src.index("float atan2_fast(float y, float x)"):]
    body = body[:body.index("\n}\n")]
    lead = float(re.search(r"float p = ([-0-9.e+]+)f;", body).group(1))
    rest = [float(v) for v in re.findall(r"p = fmaf\(p, s, ([-0-9.e+]+)f\);", body)]
    return [lead] + rest


def atan2_fast_np(y, x):
    f = np.float32
    c = [f(v) for v in _atan2_coeffs()]
    y = y.astype(f)
    x = x.astype(f)
    ax, ay = np.abs(x), np.abs(y)
    mx, mn = np.maximum(ax, ay), np.minimum(ax, ay)
    with np.errstate(divide="ignore", invalid="ignore"):
        a = (mn * (f(1) / mx)).astype(f)
    s = (a * a).astype(f)
    p = c[0]
    for ck in c[1:]:
        p = (p * s + ck).astype(f)          # fmaf: fp32 rounding of the fused result is closer still
    r = ((a * s).astype(f) * p + a).astype(f)
    r = np.where(ay > ax, ((f(1.57079637) - r).astype(f) + f(-4.37113883e-08)).astype(f), r)
    r = np.where(x < 0, ((f(3.14159274) - r).astype(f) + f(-8.74227766e-08)).astype(f), r)
    r = np.copysign(r, y)
    return np.where(mx == 0, f(0), r)


def test_atan2_fast_accuracy():
    rng = np.random.default_rng(1)
    ang = rng.uniform(-np.pi, np.pi, 400000)
    rad = np.exp(rng.uniform(-6, 6, ang.size))
    x, y = (rad * np.cos(ang)).astype(np.float32), (rad * np.sin(ang)).astype(np.float32)
    got = atan2_fast_np(y, x).astype(np.float64)
    ref = np.arctan2(y.astype(np.float64), x.astype(np.float64))
    err = got - ref
    assert np.abs(err).max() < 3e-7            # about 1 ulp of pi
    assert abs(err.mean()) < 5e-9              # no systematic bias (it would add up in P^T theta)
    small = np.abs(ref) < 1e-3                 # near the heading of a straight segment
    assert np.max(np.abs(err[small]) / np.abs(ref[small])) < 3e-7


def test_atan2_fast_special_cases():
    z = np.float32(0)
    assert atan2_fast_np(np.array([z]), np.array([z]))[0] == 0.0          # G18
    assert atan2_fast_np(np.array([np.float32(0)]), np.array([np.float32(-1)]))[0] == np.float32(np.pi)
    assert atan2_fast_np(np.array([np.float32(-0.0)]), np.array([np.float32(-1)]))[0] == -np.float32(np.pi)
    assert atan2_fast_np(np.array([np.float32(1)]), np.array([np.float32(0)]))[0] == np.float32(np.pi / 2)


def _sincos_consts():
    src = open(KERNEL).read()
    body = src[src.index("void sincos_fast(float x, float* sp, float* cp)"):]
    body = body[:body.index("\n}\n")]
    return [float(v) for v in re.findall(r"([-]?\d\.\d+e[-+]?\d+|[-]?\d\.\d{6,})f", body)]


def sincos_fast_np(x):
    """The kernel's sincos_fast in float32 numpy, constants parsed from the source in order:
    2/pi, P1, P2, P3, S3, S2, S1, C3, C2, C1."""
    f = np.float32
    k = [f(v) for v in _sincos_consts()]
    two_pi_inv, P1, P2, P3, S3, S2, S1, C3, C2, C1 = k
    x = x.astype(f)
    j = np.rint((x * two_pi_inv).astype(f)).astype(f)
    r = (x - j * abs(P1)).astype(f)
    r = (r - j * abs(P2)).astype(f)
    r = (r - j * abs(P3)).astype(f)
    r2 = (r * r).astype(f)
    sn = (r + (r * r2).astype(f) * ((S1 + r2 * ((S2 + r2 * S3).astype(f))).astype(f))).astype(f)
    cs = (f(1) - f(0.5) * r2 + (r2 * r2).astype(f) * ((C1 + r2 * ((C2 + r2 * C3).astype(f))).astype(f))).astype(f)
    q = j.astype(np.int64)
    s1, c1 = np.where(q & 1, cs, sn), np.where(q & 1, sn, cs)
    return np.where(q & 2, -s1, s1), np.where((q + 1) & 2, -c1, c1)


def test_sincos_fast_accuracy():
    assert len(_sincos_consts()) == 10
    x = np.concatenate([np.linspace(-50.0, 50.0, 400001),
                        np.random.default_rng(2).uniform(-1e3, 1e3, 100000)]).astype(np.float32)
    s, c = sincos_fast_np(x)
    xs = x.astype(np.float64)
    es, ec = s - np.sin(xs), c - np.cos(xs)
    assert np.abs(es).max() < 1.5e-7 and np.abs(ec).max() < 1.5e-7
    assert abs(es.mean()) < 1e-9 and abs(ec.mean()) < 1e-9


def test_literal_rule_offset_without_cancellation():
    """Literal-rule ellipse offset (Eq. 21a/22a with alpha = atan2(y~, x~), G8): outside
    (d* >= 1) the kernel forms a f - 1 and b f - 1 (f = N / D) as b (a - b) y~^2 / D and
    a (b - a) x~^2 / D.  Check the identity against the paper's form in fp64, and that in
    fp32 the rewritten form keeps ~1e-7 relative accuracy on nearly circular ellipses,
    where a f - 1 is a small difference of O(1) values and the direct form keeps only
    its rounding error (bmc_kernel.cuh coll_general)."""
    rng = np.random.default_rng(7)
    # the kernel's inputs are fp32 (obs_ab, x~, y~): draw them as fp32 values
    a = rng.uniform(0.4, 0.9, 2000).astype(np.float32).astype(np.float64)
    b = (a * (1.0 - rng.uniform(1e-3, 1e-2, 2000))).astype(np.float32).astype(np.float64)   # nearly circular
    ang = rng.uniform(-np.pi, np.pi, 2000)
    rho = rng.uniform(2.0, 40.0, 2000)       # outside every ellipse
    xt = (rho * np.cos(ang)).astype(np.float32).astype(np.float64)
    yt = (rho * np.sin(ang)).astype(np.float32).astype(np.float64)
    # the paper's form: delta = (a d cos(al) - x~, b d sin(al) - y~), d = max(1, d*)
    al = np.arctan2(yt, xt)
    dstar = (a * xt * np.cos(al) + b * yt * np.sin(al)) / (a**2 * np.cos(al)**2 + b**2 * np.sin(al)**2)
    d = np.maximum(dstar, 1.0)
    dx_ref, dy_ref = a * d * np.cos(al) - xt, b * d * np.sin(al) - yt
    x2, y2 = xt * xt, yt * yt
    D = a * a * x2 + b * b * y2
    assert np.all(dstar >= 1.0)
    np.testing.assert_allclose(xt * b * (a - b) * y2 / D, dx_ref, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(yt * a * (b - a) * x2 / D, dy_ref, rtol=1e-9, atol=1e-12)
    # fp32: rewritten vs direct
    f32 = np.float32
    a32, b32, x32, y32 = a.astype(f32), b.astype(f32), xt.astype(f32), yt.astype(f32)
    X2, Y2 = x32 * x32, y32 * y32
    D32 = a32 * a32 * X2 + b32 * b32 * Y2
    N32 = a32 * X2 + b32 * Y2
    rw = x32 * ((b32 * (a32 - b32)) * Y2 * (f32(1) / D32))
    direct = x32 * (a32 * (N32 / D32) - f32(1))
    big = np.abs(dx_ref) > 1e-3 * np.abs(xt) * (a - b) / a   # away from the axes
    err_rw = np.abs(rw.astype(np.float64) - dx_ref)[big] / np.abs(dx_ref[big])
    err_direct = np.abs(direct.astype(np.float64) - dx_ref)[big] / np.abs(dx_ref[big])
    assert np.median(err_rw) < 3e-7 and np.percentile(err_rw, 99) < 2e-6
    assert np.median(err_direct) > 100 * np.median(err_rw)
