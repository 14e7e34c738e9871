"""Pins of the oracle's STOMP-style sampler (oracle/sampler.c; SURVEY §8f NEXT-2, P:585,
reading G28): the Philox4x32-10 block against the published known-answer vectors, the
normals against the standard normal law, the noise covariance against STOMP's smoothness
prior computed independently (numpy), the unperturbed line and boundary points, and the
independence of an instance's sample from the batch split."""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.json")
BND = np.array([[0.0, 1.0, 0.0, 30.0, 1.0, 0.0], [0.0, 0.0, 0.0, 2.0, 0.0, 0.0], [0.0] * 6])


def test_philox_known_answers():
    for v in json.load(open(GOLD))["vectors"]:
        out = oracle.philox4x32_10([int(x, 16) for x in v["ctr"]], [int(x, 16) for x in v["key"]])
        assert out == [int(x, 16) for x in v["out"]]


def test_normals_are_standard():
    z = np.concatenate([oracle.stomp_normals(11, 0, g) for g in range(20000)])
    assert abs(z.mean()) < 0.01
    assert abs(z.var() - 1.0) < 0.01
    assert abs(np.mean(np.abs(z) < 1.0) - 0.682689) < 0.005
    assert abs(np.mean(np.abs(z) < 2.0) - 0.954500) < 0.003
    # pairs from one Box-Muller draw are uncorrelated
    zz = np.stack([oracle.stomp_normals(11, 0, g) for g in range(20000)])
    assert abs(np.corrcoef(zz[:, 0], zz[:, 1])[0, 1]) < 0.03


def stomp_prior(degree=10):
    """N(0, R^-1) on the control points 3..deg-3, R = D^T D (second difference), unit max variance."""
    nv = degree + 1
    D = np.zeros((nv - 2, nv))
    for i in range(nv - 2):
        D[i, i:i + 3] = [1.0, -2.0, 1.0]
    free = np.arange(3, nv - 3)
    S = np.linalg.inv((D.T @ D)[np.ix_(free, free)])
    return S / S.diagonal().max()


def test_factor_and_sample_covariance():
    L = oracle.stomp_factor(10)
    S = stomp_prior(10)
    assert np.allclose(L @ L.T, S, atol=1e-12)
    assert np.allclose(L, np.tril(L))
    x = oracle.sample_init(40000, BND, seed=5, sigma_x=1.0, sigma_y=2.0, line_first=False)
    line = oracle.sample_init(1, BND, seed=5, line_first=True)[0]
    ex = x[:, 0, 3:8] - line[0, 3:8]
    ey = x[:, 1, 3:8] - line[1, 3:8]
    assert np.allclose(np.cov(ex.T), S, atol=0.03)
    assert np.allclose(np.cov(ey.T), 4.0 * S, atol=0.12)
    assert np.abs(ex.mean(0)).max() < 0.02


def test_line_and_untouched_boundary_points():
    x = oracle.sample_init(64, BND, seed=9)
    k = np.arange(11) / 10
    line_x, line_y = 30.0 * k, 2.0 * k
    assert np.array_equal(x[0, 0], line_x) and np.array_equal(x[0, 1], line_y)   # instance 0: the line
    for idx in (0, 1, 2, 8, 9, 10):                 # p, v, a at both ends stay those of the line
        assert np.allclose(x[:, 0, idx], line_x[idx]) and np.allclose(x[:, 1, idx], line_y[idx])
    assert np.all(x[:, 2] == 0.0)
    assert np.std(x[1:, 1, 5]) > 0.5


@pytest.mark.parametrize("split", [1, 7, 33])
def test_samples_do_not_depend_on_the_batch_split(split):
    full = oracle.sample_init(100, BND, seed=3, stream=17)
    part = oracle.sample_init(100 - split, BND, seed=3, stream=17, index_base=split)
    assert np.array_equal(full[split:], part)
    other = oracle.sample_init(100, BND, seed=3, stream=18)
    assert not np.allclose(full[1:], other[1:])       # another stream, other samples
