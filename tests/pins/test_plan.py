"""Pins for oracle/plan.py against closed forms (Eq. (1), Eq. (4))."""
import math

import numpy as np
import pytest

from oracle import plan
from tests.conftest import golden_lines


def _golden_eigen():
    out = {}
    for ln in golden_lines("eigen_closed_forms.txt"):
        name, C, lam, alpha = [s.strip() for s in ln.split("|")]
        C = np.array([float(x) for x in C.split()])
        d = int(round(math.sqrt(C.size)))
        out[name] = (C.reshape(d, d), np.array([float(x) for x in lam.split()]),
                     np.array([float(x) for x in alpha.split()]))
    return out


@pytest.mark.parametrize("name", ["spec_2x2", "cfg3"])
def test_diagonalize_closed_forms(name):
    C, lam, alpha = _golden_eigen()[name]
    Q, a = plan.diagonalize(C)
    np.testing.assert_allclose(a, alpha, rtol=1e-8)
    np.testing.assert_allclose(Q.T @ Q, np.eye(len(a)), atol=1e-12)
    np.testing.assert_allclose(Q @ np.diag(a ** 2) @ Q.T, np.linalg.inv(C), rtol=1e-10,
                               atol=1e-12 * np.abs(np.linalg.inv(C)).max())
    # each column is an eigenvector of C with eigenvalue 1/alpha^2
    for k in range(len(a)):
        np.testing.assert_allclose(C @ Q[:, k], Q[:, k] / a[k] ** 2, rtol=1e-9, atol=1e-9)


def test_cfg3_middle_eigenvector_closed_form():
    C, _, _ = _golden_eigen()["cfg3"]
    Q, _ = plan.diagonalize(C)
    # (1, 0, -1)/sqrt2 with eigenvalue 0.7*35^2, sign convention: first component positive
    np.testing.assert_allclose(Q[:, 1], np.array([1, 0, -1]) / math.sqrt(2), atol=1e-12)


def test_diagonal_c_is_identity_no_reorder():
    C = np.diag([4.0, 9.0, 1.0])
    Q, a = plan.diagonalize(C)
    assert np.array_equal(Q, np.eye(3))
    np.testing.assert_allclose(a, [0.5, 1 / 3, 1.0])


def test_random_spd_invariants_and_quadratic_form():
    rng = np.random.default_rng(0)
    for d in (2, 3, 5, 8):
        A = rng.normal(size=(d, d))
        C = A @ A.T + d * np.eye(d)
        Q, a = plan.diagonalize(C)
        assert np.all(np.diff(a) <= 1e-15)            # alpha descending
        x = rng.normal(size=d) * 20
        y = Q.T @ x
        np.testing.assert_allclose(np.sum(a ** 2 * y ** 2), x @ np.linalg.solve(C, x), rtol=1e-10)
        for k in range(d):
            col = Q[:, k]
            first = np.nonzero(np.abs(col) > 1e-6 * np.abs(col).max())[0][0]
            assert col[first] > 0


def test_diagonalize_errors():
    with pytest.raises(ValueError):
        plan.diagonalize(np.array([[1.0, 0.5], [0.4, 1.0]]))
    with pytest.raises(ValueError):
        plan.diagonalize(np.array([[1.0, 2.0], [2.0, 1.0]]))


def test_taps_closed_form():
    for s in (0.7, 1.0, 2.0, 5.0, 16.0):
        r = plan.radius(s)
        assert r == math.ceil(3 * s)
        w = plan.spatial_taps(s)
        assert w.shape == (2 * r + 1,)
        assert abs(w.sum() - 1.0) < 1e-15
        np.testing.assert_array_equal(w, w[::-1])
        for m in range(-r, r + 1):
            assert abs(w[m + r] / w[r] - math.exp(-m * m / (2 * s * s))) < 1e-15


def test_gammas():
    np.testing.assert_allclose(plan.gammas([0.1, 0.2], 25), [0.02, 0.04], rtol=1e-15)
