"""Pins of the scheme-solver oracle (oracle/solver.py) against what
the paper / its specification fix: worked examples, the ratio
properties of the closed forms, Lagrange stationarity checked
numerically (not by retyping the formula), constraint satisfaction after rounding,
and exhaustive integer searches on small problems."""
import numpy as np
import pytest

from oracle import solver


def test_predict_error_worked_example():
    """H = 1, Delta = 0.1, g = 12 -> E[dz] = 0.01, sigma_pred = 0.1; all
    Delta = 0 -> 0."""
    assert solver.predict_error([0.1], [12.0]) == pytest.approx(0.1, rel=1e-15)
    assert solver.predict_error([0.0, 0.0], [3.0, 5.0]) == 0.0


def test_error_bounded_worked_example():
    """H = 1, P = 1000, g = 4, z = 10, eps = 0.01, R = 1 -> Delta = sqrt(0.03)
    = 0.17321, b = ceil(2.529) = 3."""
    d, b = solver.solve_error_bounded([1000.0], [4.0], [1.0], 10.0, 0.01)
    assert d[0] == pytest.approx(0.17320508075688773, rel=1e-14)
    assert b[0] == 3


def test_error_bounded_gradient_ratio_gives_one_bit():
    """P_1 = P_2, g_2 = 4 g_1 -> Delta_2 = Delta_1 / 2: exactly one more fraction
    bit on quantity 2 before the ceiling."""
    d, b = solver.solve_error_bounded([500.0, 500.0], [3.0, 12.0], [2.0, 2.0], 7.0, 0.02)
    assert d[1] == pytest.approx(d[0] / 2, rel=1e-14)
    assert -np.log2(d[1] / 2.0) == pytest.approx(-np.log2(d[0] / 2.0) + 1.0, abs=1e-12)


@pytest.mark.parametrize("seed", range(5))
def test_error_bounded_is_the_constrained_optimum(seed):
    """Lagrange stationarity of Eq. 9 checked numerically: the continuous Delta meets
    the error constraint with equality, and every feasible move along the constraint
    surface (two coordinates traded against each other) raises the bit count."""
    rng = np.random.default_rng(seed)
    H = 4
    P = rng.uniform(1e2, 1e4, H)
    g = rng.uniform(0.1, 10.0, H)
    R = 2.0 ** rng.integers(-2, 6, H)
    z, eps = 3.0, 0.05
    d = solver.error_bounded_delta(P, g, z, eps)
    assert np.sum(d * d * g) / 12.0 == pytest.approx((eps * z) ** 2, rel=1e-12)
    cost = lambda dd: float(np.sum(-P * np.log2(dd / R)))
    c0 = cost(d)
    for i in range(H):
        for j in range(H):
            if i == j:
                continue
            for s in (0.9, 0.97, 1.03, 1.1):
                dd = d.copy()
                dd[i] *= s  # keep sum d^2 g fixed by adjusting j
                rest = (d[i] ** 2 - dd[i] ** 2) * g[i] + d[j] ** 2 * g[j]
                if rest <= 0:
                    continue
                dd[j] = np.sqrt(rest / g[j])
                assert cost(dd) > c0 - 1e-9


@pytest.mark.parametrize("seed", range(6))
def test_error_bounded_ceiling_keeps_the_bound_and_is_near_optimal(seed):
    """Algorithm 1 line 15 (ceiling) only shrinks Delta, so sigma_pred <= eps |z|
    (S:335); an exhaustive search over integer bit vectors finds at most H fewer
    total fraction bits (at most one bit per type)."""
    rng = np.random.default_rng(100 + seed)
    H = 3
    P = rng.integers(1, 10, H).astype(np.float64)
    g = rng.uniform(0.05, 20.0, H)
    R = 2.0 ** rng.integers(-1, 4, H)
    z, eps = 2.0, 0.01
    d, b = solver.solve_error_bounded(P, g, R, z, eps, b_max=20)
    dq = solver.bits_to_delta(b, R)
    assert np.all(dq <= d * (1 + 1e-12))
    assert solver.predict_error(dq, g) <= eps * abs(z) * (1 + 1e-12)
    best, bb = solver.brute_force_error_bounded(P, g, R, z, eps, b_max=20)
    assert np.dot(P, b) <= best + np.sum(P)  # <= one bit per variable of each type


def test_error_bounded_zero_gradient_gets_b_min():
    """S:337 errors: a quantity with g_h = 0 bypasses the formula (b = b_min)."""
    d, b = solver.solve_error_bounded([10.0, 10.0], [0.0, 2.0], [1.0, 1.0], 1.0, 0.1, b_min=2)
    assert b[0] == 2 and np.isinf(d[0]) and b[1] >= 2


def test_memory_bounded_symmetric_split():
    """H = 2, P_1 = P_2, g_1 = g_2, R_1 = R_2, 20 fraction bits per pair ->
    b = (10, 10)."""
    d, b = solver.solve_memory_bounded([1.0, 1.0], [3.0, 3.0], [4.0, 4.0], 20.0)
    assert list(b) == [10, 10]
    assert d[0] == pytest.approx(4.0 * 2.0 ** -10, rel=1e-12)


def test_memory_bounded_gradient_ratio_moves_half_a_bit():
    """doubling g_2 (all else equal) moves exactly half a bit of precision to
    quantity 2 before flooring: log2(Delta_1 / Delta_2) = 1/2."""
    d, _ = solver.solve_memory_bounded([5.0, 5.0], [1.0, 2.0], [1.0, 1.0], 80.0)
    assert np.log2(d[0] / d[1]) == pytest.approx(0.5, abs=1e-12)


@pytest.mark.parametrize("seed", range(6))
def test_memory_bounded_meets_budget_and_is_near_optimal(seed):
    """The floor keeps the budget hard; versus an exhaustive search the predicted error
    is within a factor 4 of the integer optimum (flooring costs at most about a
    bit per type, 2x on Delta)."""
    rng = np.random.default_rng(200 + seed)
    H = 3
    P = rng.integers(1, 8, H).astype(np.float64)
    g = rng.uniform(0.05, 20.0, H)
    R = 2.0 ** rng.integers(-1, 4, H)
    B = float(rng.integers(15, 45)) * P.mean()
    d, b = solver.solve_memory_bounded(P, g, R, B, b_max=20)
    assert np.dot(P, b) <= B
    err = solver.predict_error(solver.bits_to_delta(b, R), g)
    best, _ = solver.brute_force_memory_bounded(P, g, R, B, b_max=20)
    assert err <= 4.0 * best * (1 + 1e-12)


def test_memory_bounded_infeasible_budget():
    with pytest.raises(ValueError):
        solver.solve_memory_bounded([10.0, 10.0], [1.0, 1.0], [1.0, 1.0], 30.0, b_min=2)


def test_memory_bounded_active_set_refits_clamped_widths():
    """A type the closed form puts below b_min is fixed there and the others re-solved with
    the budget it leaves: P = (1, 1), g = (1e-12, 1), R = 1, B = 10, b_min = 3
    -> the first type takes 3, the second the remaining 7 (the one-shot form gave the
    second 16 bits and broke the budget)."""
    d, b = solver.solve_memory_bounded([1.0, 1.0], [1e-12, 1.0], [1.0, 1.0], 10.0, b_min=3)
    assert list(b) == [3, 7] and np.dot([1.0, 1.0], b) <= 10.0


@pytest.mark.parametrize("seed", range(6))
def test_memory_bounded_with_clamps_near_optimal(seed):
    """Gradients over 11 orders of magnitude force widths onto both box bounds; the
    active-set scheme meets the budget and stays within 4x of the exhaustive optimum's
    predicted error."""
    rng = np.random.default_rng(300 + seed)
    H = 3
    P = rng.integers(1, 8, H).astype(np.float64)
    g = 10.0 ** rng.uniform(-8, 3, H)
    R = 2.0 ** rng.integers(-1, 4, H)
    B = float(rng.integers(10, 40)) * P.mean()
    d, b = solver.solve_memory_bounded(P, g, R, B, b_min=0, b_max=12)
    assert np.dot(P, b) <= B and b.min() >= 0 and b.max() <= 12
    err = solver.predict_error(solver.bits_to_delta(b, R), g)
    best, _ = solver.brute_force_memory_bounded(P, g, R, B, b_max=12)
    assert err <= 4.0 * best * (1 + 1e-12)
