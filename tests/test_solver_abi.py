"""The library's scheme solver (qmpm_solve_*, qmpm_predict_error: host code behind the
C ABI, no GPU) against the solver oracle (oracle/solver.py) on random problems."""
import numpy as np
import pytest

from oracle import solver as osol
from paper_2207_04658_b200 import qmpm


@pytest.mark.parametrize("seed", range(8))
def test_error_bounded_matches_oracle(seed):
    rng = np.random.default_rng(seed)
    H = int(rng.integers(1, 30))
    P = rng.integers(1, 10 ** 6, H).astype(np.float64)
    g = rng.uniform(0.0, 50.0, H) * (rng.uniform(size=H) > 0.1)
    R = 2.0 ** rng.integers(-4, 8, H)
    z, eps = float(rng.uniform(0.1, 100)), float(10.0 ** rng.uniform(-4, -1))
    d, b = qmpm.solve_error_bounded(P, g, R, z, eps, b_min=1, b_max=30)
    do, bo = osol.solve_error_bounded(P, g, R, z, eps, b_min=1, b_max=30)
    assert list(b) == list(bo)
    fin = np.isfinite(do)
    np.testing.assert_allclose(d[fin], do[fin], rtol=1e-13)
    assert np.all(np.isinf(d[~fin]))
    assert qmpm.predict_error(osol.bits_to_delta(b, R), g) == pytest.approx(
        osol.predict_error(osol.bits_to_delta(bo, R), g), rel=1e-13)


@pytest.mark.parametrize("seed", range(8))
def test_memory_bounded_matches_oracle(seed):
    rng = np.random.default_rng(50 + seed)
    H = int(rng.integers(1, 30))
    P = rng.integers(1, 10 ** 6, H).astype(np.float64)
    g = rng.uniform(0.0, 50.0, H) * (rng.uniform(size=H) > 0.1)
    R = 2.0 ** rng.integers(-4, 8, H)
    B = float(rng.uniform(4, 24)) * P.sum()
    d, b = qmpm.solve_memory_bounded(P, g, R, B, b_min=2, b_max=30)
    do, bo = osol.solve_memory_bounded(P, g, R, B, b_min=2, b_max=30)
    assert list(b) == list(bo)
    fin = np.isfinite(do)
    np.testing.assert_allclose(d[fin], do[fin], rtol=1e-12)
    assert np.dot(P, b) <= B


def test_solver_rejects_bad_input():
    with pytest.raises(qmpm.QmpmError):
        qmpm.solve_error_bounded([1.0], [1.0], [0.0], 1.0, 0.1)  # R = 0
    with pytest.raises(qmpm.QmpmError):
        qmpm.solve_error_bounded([1.0], [1.0], [1.0], 0.0, 0.1)  # z = 0
    with pytest.raises(qmpm.QmpmError):
        qmpm.solve_memory_bounded([10.0, 10.0], [1.0, 1.0], [1.0, 1.0], 30.0, b_min=2)  # infeasible
    with pytest.raises(qmpm.QmpmError):
        qmpm.solve_error_bounded([1.0], [-1.0], [1.0], 1.0, 0.1)  # g < 0


def test_error_bounded_reports_an_unmet_bound():
    """With b_max too small for eps the library returns QMPM_EDOMAIN (the clamped scheme
    still filled: strict=False) instead of silently missing the bound."""
    P, g, R = [100.0, 100.0], [50.0, 2.0], [4.0, 4.0]
    with pytest.raises(qmpm.QmpmError):
        qmpm.solve_error_bounded(P, g, R, 1.0, 1e-4, b_min=0, b_max=6)
    d, b = qmpm.solve_error_bounded(P, g, R, 1.0, 1e-4, b_min=0, b_max=6, strict=False)
    assert list(b) == [6, 6]
    d, b = qmpm.solve_error_bounded(P, g, R, 1.0, 1e-4, b_min=0, b_max=30)
    assert qmpm.predict_error(osol.bits_to_delta(b, R), g) <= 1e-4


def test_memory_bounded_refits_clamped_widths():
    d, b = qmpm.solve_memory_bounded([1.0, 1.0], [1e-12, 1.0], [1.0, 1.0], 10.0, b_min=3)
    assert list(b) == [3, 7]
